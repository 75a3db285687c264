# scratch GPU job: blend A/B (fast SFU path vs GSC_F_BLEND_EXACT) on the same box, 300 C4 frames each, twice
mkdir -p gpurun_out/$1
for V in "" "--blend-exact" "" "--blend-exact"; do
timeout 400 python bench.py --steps 300 --warmup 5 --no-cpu-baseline $V > gpurun_out/$1/b.txt 2>&1
tail -1 gpurun_out/$1/b.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$V', d['value'], d['serial_ms_per_frame'], {k:v['ms_per_frame'] for k,v in d['stages'].items() if k in ('blend',)}, d['frame_counts']['evals'])"
done
