T=tools/tma_bw
for m in 1 2; do for br in 64 128 256 512; do $T $m 1 $br 6 512; done; done
$T 2 148 128 11 1024; $T 1 148 128 11 1024; $T 2 148 256 6 1024
