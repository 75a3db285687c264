# scratch GPU job: ncu --set full of every kernel of one frame: $2 = frame index in the timed pass (18 launches/frame)
mkdir -p gpurun_out/$1
F=${2:-10}
timeout 900 ncu --set full --clock-control none --import-source on -s $(( (F + 3) * 18 )) -c 18 -o gpurun_out/$1/frame$F python bench.py --steps $((F + 2)) --warmup 3 --no-cpu-baseline > gpurun_out/$1/ncu_full.txt 2>&1
tail -2 gpurun_out/$1/ncu_full.txt
