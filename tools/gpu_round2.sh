#!/bin/bash
# Round-2 measurement on one B200: GPU tests, smoke, bench (ours + 2-rank
# gloo), launch list, ncu --set full of the reduction kernels, per-group solve
# profiles.  Outputs under gpurun_out/$TAG/.  TESTS=0 skips the test suite.
set -x
TAG=${TAG:-r2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $OUT/smi.txt
if [ "${TESTS:-1}" = 1 ]; then
  timeout 1200 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.txt 2>&1
  timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.txt 2>&1
fi
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --gpus 2 --comm gloo --no-cpu-baseline > $OUT/bench_g2.json 2> $OUT/bench_g2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches_1354.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-runs 1 > /dev/null 2>&1
for c in "case1354pegase 256" "case1354pegase 32" "case2869pegase 512" "case118 64"; do
  set -- $c
  timeout 900 python tools/profile_solve.py $1 $2 > $OUT/profile_$1_N$2.json 2>&1
done
timeout 900 python tools/profile_solve.py case9241pegase 128 0.05 3 > $OUT/profile_case9241pegase_N128.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"reduce_stream|reach_solve|gemm_tn|xt_sparse" -c 4 -o $OUT/ncu_reduce_1354 python tools/micro_reduce.py case1354pegase 256 1 > $OUT/ncu_reduce.log 2>&1
ls -la $OUT
