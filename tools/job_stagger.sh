# scratch GPU job: staggered-expiry parity + C4 bench with and without it
mkdir -p gpurun_out/$1
timeout 600 python -m pytest tests -x -q -m gpu -k "stagger or c1_all_poses or c1_moving or c4_full or guide" > gpurun_out/$1/pytest_gpu.txt 2>&1
tail -2 gpurun_out/$1/pytest_gpu.txt
for V in "" "--stagger"; do
timeout 400 python bench.py --steps 600 --warmup 5 --no-cpu-baseline $V > gpurun_out/$1/bench_C4$V.txt 2>&1
tail -1 gpurun_out/$1/bench_C4$V.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['frame_ms'], {k:v['ms_per_frame'] for k,v in d['stages'].items()})"
done
