for st in 10 5; do for sk in 0 1 2 8 11 13 15; do echo "== stages $st skip $sk"; python tools/decode_probe.py --ticks 32 --repeat 2 --stages $st --skip $sk 2>&1 | tail -1; done; done
echo "== no pdl"; python tools/decode_probe.py --ticks 32 --repeat 2 --pdl 0 | tail -1
echo "== no graphs"; python tools/decode_probe.py --ticks 32 --repeat 2 --graphs 0 | tail -1
echo "== rows 1"; python tools/decode_probe.py --ticks 32 --repeat 2 --rows 1 | tail -1
