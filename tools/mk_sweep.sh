# chunk-plan sweep of the persistent decode-tick kernel (tools/decode_probe.py)
for cfg in "--opt mk_nc_cap=8" "--opt mk_nc_cap=6" "--opt mk_nc_cap=4" "--opt mk_nc_cap=8 --opt mk_per_cta=5" "--opt mk_nc_cap=8 --opt mk_nc_cap_o=16" "--opt mk_nc_cap=6 --opt mk_nc_cap_o=8"; do
  echo "== $cfg"; timeout 100 python tools/decode_probe.py --ticks 32 --repeat 3 $cfg 2>&1 | tail -1 | cut -c40-90
done
