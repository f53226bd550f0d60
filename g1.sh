mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
for c in 0 1 2 4; do python bench.py --config $c --steps 20 --warmup 3 --no-cpu > gpurun_out/b$c.json 2>gpurun_out/b$c.err; python -c "import json,sys; d=json.loads(open('gpurun_out/b$c.json').read()); print(d['config']['workload'][:3], round(d['ms_per_step'],4), round(d['value'],1), {k:round(v,4) for k,v in d.get('kernel_ms').items()})"; done
