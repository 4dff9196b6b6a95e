#!/bin/bash
# ncu full captures of the dense / attention kernels and compute-sanitizer
# runs (run under gpurun; outputs land in gpurun_out/, summaries go to
# profiles/ via tools/ncu_full_summary.py).
set -u
O=gpurun_out
P="python tools/decode_probe.py --repeat 1"
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 $NCU -k regex:gemm_pair -s 1 -c 3 -o $O/ncu_pair -f $P --ticks 1 > $O/ncu_pair.log 2>&1; echo "pair rc=$?"
timeout 300 $NCU -k regex:prefill_attn -s 1 -c 1 -o $O/ncu_pattn -f $P --ticks 1 > $O/ncu_pattn.log 2>&1; echo "pattn rc=$?"
timeout 300 $NCU -k regex:vattn_bf16 -s 2 -c 1 -o $O/ncu_vattn -f python tools/vision_probe.py > $O/ncu_vattn.log 2>&1; echo "vattn rc=$?"
timeout 300 $NCU -k regex:attn_span -s 40 -c 1 -o $O/ncu_span64 -f python tools/span_probe.py --config 7b --episodes 64 --tokens 3 > $O/ncu_span64.log 2>&1; echo "span64 rc=$?"
timeout 300 $NCU -k regex:attn_span -s 64 -c 1 -o $O/ncu_span -f $P --rows 24 --ticks 3 > $O/ncu_span.log 2>&1; echo "span rc=$?"
timeout 300 $NCU -k regex:decode_mk -s 1 -c 1 -o $O/ncu_tick -f $P --ticks 3 > $O/ncu_tick.log 2>&1; echo "tick rc=$?"
timeout 900 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 \
  python -m pytest tests/test_engine_gpu.py -x -q -k "bit_exact or fork_cow or gemm_tc_matches or span_attention_matches_page_items and small or vision or tag_in_prefill or draft or batched_prefill and tiny or prefill_tensor_core" \
  > $O/sanitizer_memcheck.log 2>&1; echo "memcheck rc=$?"
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 \
  python -m pytest tests/test_engine_gpu.py -x -q -k "test_request_tokens_and_logits_bit_exact or test_gemm_tc_matches_torch" \
  > $O/sanitizer_racecheck.log 2>&1; echo "racecheck rc=$?"
tail -n 3 $O/sanitizer_memcheck.log; tail -n 3 $O/sanitizer_racecheck.log
