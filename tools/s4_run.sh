sh tools/ab_bench.sh "libjsontape_b200 ab_t128 ab_t128b" "4 1" > gpurun_out/s4_ab1.txt 2>&1
cat gpurun_out/s4_ab1.txt
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name 'regex:k_index|k_stage1' -c 2 -f -o gpurun_out/s4_src_c4 python tools/prof.py --config 4 --size 268435456 --reps 1 > gpurun_out/s4_ncu.log 2>&1
tail -3 gpurun_out/s4_ncu.log
