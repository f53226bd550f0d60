for r in 1 2; do
for v in A B; do
if [ $v = A ]; then export JT_B200_LIB=$PWD/exp/libA.so; else unset JT_B200_LIB; fi
python bench.py --config 1 --steps 20 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), round(d['kernel_ms']['struct'],4))"
done; done
