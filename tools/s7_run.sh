#!/bin/bash
# End-of-session evidence run on the GPU box: the GPU test suite, the default bench and the
# reference arm, the launch list of the headline command and the ncu --set full captures the
# summaries under profiles/ are made from (tools/ncu_summary.py).
mkdir -p gpurun_out
( time python -m pytest tests -m gpu -x -q ) > gpurun_out/s10_gputests.log 2>&1
python bench.py > gpurun_out/s10_bench.json 2> gpurun_out/s10_bench.err
python bench.py --impl reference > gpurun_out/s10_bench_ref.json 2> gpurun_out/s10_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/s10_launches_bench_c4.csv python bench.py --no-table --no-cpu --steps 2 --warmup 3 > gpurun_out/s10_ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -c 40 -o gpurun_out/s10_full_c4 -f python tools/prof.py --config 4 --mode both --reps 1 > gpurun_out/s10_ncu_c4.log 2>&1
ncu --set full --clock-control none --import-source on -c 40 -o gpurun_out/s10_full_c1 -f python tools/prof.py --config 1 --mode both --reps 1 > gpurun_out/s10_ncu_c1.log 2>&1
tail -3 gpurun_out/s10_gputests.log
head -c 300 gpurun_out/s10_bench.json
