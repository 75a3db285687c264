# scratch GPU job: C4 bench (300 frames) + optional launch list of kernels matching $2
mkdir -p gpurun_out/$1
timeout 400 python bench.py --steps 300 --warmup 5 --no-cpu-baseline > gpurun_out/$1/bench_C4.txt 2>&1
tail -1 gpurun_out/$1/bench_C4.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['serial_ms_per_frame'], d['frame_counts']['blend_fixup_pixels']); print({k:v['ms_per_frame'] for k,v in d['stages'].items()})"
if [ -n "$2" ]; then
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:$2" -s ${3:-200} -c ${4:-60} --csv --log-file gpurun_out/$1/launches.csv python bench.py --steps 60 --warmup 3 --no-cpu-baseline > gpurun_out/$1/ncu1.txt 2>&1
python tools/ncu_launch_summary.py gpurun_out/$1/launches.csv
fi
