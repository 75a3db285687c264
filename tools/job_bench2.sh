# scratch GPU job: C4 bench lines, 600 and 20 frames
mkdir -p gpurun_out/$1
for S in 600 20; do
timeout 600 python bench.py --steps $S --warmup 5 --no-cpu-baseline > gpurun_out/$1/bench_$S.txt 2>&1
tail -1 gpurun_out/$1/bench_$S.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($S, d['value'], d['e2e']['value'], d['roofline']['frac'], d['serial_ms_per_frame'], {k:v['ms_per_frame'] for k,v in d['stages'].items()})"
done
