#!/bin/bash
# end-of-round measurement: bench (ours + 2-rank gloo), launch list, ncu
# summaries (reports summarised on the box; they stay there)
OUT=${OUTF:-gpurun_out/final}
mkdir -p $OUT
T=/tmp/ncuf; mkdir -p $T
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $OUT/smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.txt 2>&1
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --gpus 2 --comm gloo --no-cpu-baseline > $OUT/bench_g2.json 2> $OUT/bench_g2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches_1354.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-runs 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"reduce_stream|reach_solve|gemm_tn|xt_sparse" -c 4 -o $T/reduce_1354 python tools/micro_reduce.py case1354pegase 256 1 > $OUT/ncu_reduce.log 2>&1
python tools/ncu_summarize.py report $T/reduce_1354.ncu-rep $OUT/ncu_reduce_1354.json > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"ad_|condense|transpose_in|refactor|reduce_rhs|recover_state|cholesky|blocked_solve|pad_dense|gemm_nn" -c 60 -o $T/small_1354 python tools/profile_solve.py case1354pegase 256 0.05 2 > $OUT/ncu_small.log 2>&1
python tools/ncu_summarize.py report $T/small_1354.ncu-rep $OUT/ncu_small_1354.json > /dev/null 2>&1
ls -la $OUT
