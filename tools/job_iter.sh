# scratch GPU iteration job: parity subset, short bench (stage ms), sort/emit launch durations
mkdir -p gpurun_out/$1
timeout 500 python -m pytest tests -x -q -m gpu -k "c1_all_poses or c1_moving or c3_trajectory or c4_full or reset_and_empty" > gpurun_out/$1/pytest_gpu.txt 2>&1
tail -2 gpurun_out/$1/pytest_gpu.txt
timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu-baseline > gpurun_out/$1/bench_C4.txt 2>&1
tail -1 gpurun_out/$1/bench_C4.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], {k:v['ms_per_frame'] for k,v in d['stages'].items()})"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:${2:-sweep|spine|onesweep}" -s 1800 -c 180 --csv --log-file gpurun_out/$1/launches.csv python bench.py --steps 120 --warmup 3 --no-cpu-baseline > gpurun_out/$1/ncu1.txt 2>&1
python tools/ncu_launch_summary.py gpurun_out/$1/launches.csv
