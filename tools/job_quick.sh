# scratch GPU job: a pytest -k subset ($2) and one C4 bench line ($3 steps)
mkdir -p gpurun_out/$1
timeout 1200 python -m pytest tests -x -q -m gpu -k "$2" > gpurun_out/$1/pytest_gpu.txt 2>&1
tail -3 gpurun_out/$1/pytest_gpu.txt
timeout 600 python bench.py --steps ${3:-600} --warmup 5 --no-cpu-baseline > gpurun_out/$1/bench_C4.txt 2>&1
tail -1 gpurun_out/$1/bench_C4.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline'].get('frac_executed'), d['serial_ms_per_frame'], d['frame_counts']); print({k:v['ms_per_frame'] for k,v in d['stages'].items()})"
