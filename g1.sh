mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:"k_scalars|k_struct|k_stack|k_numbers" -s 4 -c 4 -o gpurun_out/k2 -f python bench.py --config 1 --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu.log 2>&1; tail -1 gpurun_out/ncu.log
