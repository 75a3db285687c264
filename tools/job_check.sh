# scratch GPU job: full GPU tests, C4 bench (300 frames), blend/fixup launch list.  Outputs gpurun_out/$1/
mkdir -p gpurun_out/$1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$1/smoke.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/$1/pytest_gpu.txt 2>&1
tail -3 gpurun_out/$1/pytest_gpu.txt
timeout 400 python bench.py --steps 300 --warmup 5 --no-cpu-baseline > gpurun_out/$1/bench_C4.txt 2>&1
tail -1 gpurun_out/$1/bench_C4.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['frame_counts']); print({k:v['ms_per_frame'] for k,v in d['stages'].items()})"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:${2:-blend}" -s 200 -c 60 --csv --log-file gpurun_out/$1/launches.csv python bench.py --steps 60 --warmup 3 --no-cpu-baseline > gpurun_out/$1/ncu1.txt 2>&1
python tools/ncu_launch_summary.py gpurun_out/$1/launches.csv
