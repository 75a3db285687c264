# scratch GPU job: A/B of an experiment env switch ($2=VAR) on parity subset + C4 bench (300 frames)
mkdir -p gpurun_out/$1
export $2=1; timeout 500 python -m pytest tests -x -q -m gpu -k "c1_all_poses or c1_moving or c3_trajectory or c4_full" > gpurun_out/$1/pytest_gpu.txt 2>&1; unset $2
tail -2 gpurun_out/$1/pytest_gpu.txt
for V in 0 1 0 1; do
env $2=$V timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu-baseline > gpurun_out/$1/b$V.txt 2>&1
tail -1 gpurun_out/$1/b$V.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2=$V', d['value'], {k:v['ms_per_frame'] for k,v in d['stages'].items() if 'sort' in k})"
done
