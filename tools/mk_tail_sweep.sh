# fine-chunk tail sweep of the persistent decode-tick kernel (options mk_tail / mk_tail_nc)
for cfg in "--opt mk_tail=0" "--opt mk_tail=148" "--opt mk_tail=296" "--opt mk_tail=148 --opt mk_tail_nc=12" "--opt mk_tail=444" "--opt mk_tail=296 --opt mk_per_cta=3" "--opt mk_tail=148 --opt mk_per_cta=3"; do
  echo "== $cfg"; timeout 100 python tools/decode_probe.py --ticks 32 --repeat 3 $cfg 2>&1 | tail -1 | cut -c40-100
done
