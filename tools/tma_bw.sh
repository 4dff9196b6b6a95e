# weight-streaming microbenchmark sweep (tools/tma_bw.cu)
T=tools/tma_bw
for m in 0 1; do
  for g in 1 16 148; do $T $m $g 128 11 1024; done
  for s in 4 8 16; do $T $m 148 128 $s 1024; done
  $T $m 148 64 22 1024; $T $m 148 256 6 1024
  $T $m 148 128 11 32   # L2-resident pass
done
