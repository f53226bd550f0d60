mkdir -p gpurun_out
python bench.py --config 1 --steps 20 --warmup 3 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_c1.csv python bench.py --config 1 --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_stage1|k_carry_fn|k_scalars|k_numbers|k_struct|k_stack" -s 9 -c 7 -o gpurun_out/full_c1 -f python bench.py --config 1 --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
