#!/bin/bash
# Round measurement on one B200: tests, bench (default config), launch list and
# one full ncu capture of the dominant kernel.  Outputs under gpurun_out/.
set -x
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $OUT/smi.txt
timeout 600 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.txt 2>&1
timeout 300 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 300 python bench.py --case case1354pegase --scenarios 256 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench1354.json 2> $OUT/bench1354.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/launches_118.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:reduce_tiles -s 4 -c 2 -o $OUT/prof_reduce_118 -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu118.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:reduce_tiles -s 2 -c 1 -o $OUT/prof_reduce_1354 -f python bench.py --case case1354pegase --scenarios 256 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu1354.log 2>&1
ls -la $OUT
