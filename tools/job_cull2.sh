# scratch GPU job: parity subset + cull at 18M + short bench
mkdir -p gpurun_out/$1
timeout 1200 python -m pytest tests -x -q -m gpu -k "c1_all or c3_trajectory or c4_full or stagger or guide or cold or c5 or reset" > gpurun_out/$1/pytest_gpu.txt 2>&1
tail -3 gpurun_out/$1/pytest_gpu.txt
timeout 900 python tools/cull_scale.py 18000000 30 gpurun_out/$1/cull_18M.json > gpurun_out/$1/cull.txt 2>&1; tail -1 gpurun_out/$1/cull.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/$1/bench_C4.txt 2>&1
tail -1 gpurun_out/$1/bench_C4.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['roofline']['frac'], {k:v['ms_per_frame'] for k,v in d['stages'].items()})"
