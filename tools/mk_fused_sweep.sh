# fused-reduction mask sweep of the persistent decode-tick kernel
# bits: 1 QKV, 2 O, 4 gate/up, 8 down, 16 lm_head (always fused)
for f in 20 16 21 22 28 31 30; do
  echo "== mk_fused=$f"; timeout 100 python tools/decode_probe.py --ticks 32 --repeat 3 --opt mk_fused=$f 2>&1 | tail -1 | cut -c40-100
done
