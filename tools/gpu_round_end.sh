#!/bin/bash
# End-of-round measurement on one B200 (round 2): GPU tests, reduction
# micro-benchmarks, full-solve profiles, then bench (ours + 2-rank gloo),
# launch list and ncu summaries (reports summarised on the box).
# Usage: gpurun -- bash tools/gpu_round_end.sh   (outputs under gpurun_out/end, gpurun_out/final)
OUT=gpurun_out/end
mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.txt 2>&1
for cfg in "case1354pegase 256" "case2869pegase 512" "case9241pegase 128" "case1354pegase 32"; do
  echo "== $cfg" >> $OUT/micro.txt
  timeout 300 python tools/micro_reduce.py $cfg 3 2>&1 | head -1 >> $OUT/micro.txt
done
for c in "case1354pegase 256" "case1354pegase 32" "case2869pegase 512" "case118 64"; do
  set -- $c
  timeout 900 python tools/profile_solve.py $1 $2 > $OUT/profile_$1_N$2.json 2>&1
done
timeout 900 python tools/profile_solve.py case9241pegase 128 0.05 3 > $OUT/profile_case9241pegase_N128.json 2>&1
bash tools/gpu_final.sh
