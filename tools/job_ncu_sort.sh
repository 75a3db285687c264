# scratch GPU job: ncu --set full (source view) of one frame's onesweep passes (depth x4, tile x2), frame ~20
mkdir -p gpurun_out/$1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:onesweep -s $((6 * 23)) -c 6 -o gpurun_out/$1/sort python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/$1/ncu.txt 2>&1
tail -2 gpurun_out/$1/ncu.txt
