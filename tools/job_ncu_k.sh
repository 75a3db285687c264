# scratch GPU job: ncu --set full (source view) of kernels matching regex $2 at launch skip $3 (count $4)
mkdir -p gpurun_out/$1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$2" -s ${3:-20} -c ${4:-1} -o gpurun_out/$1/k python bench.py --steps 40 --warmup 3 --no-cpu-baseline > gpurun_out/$1/ncu.txt 2>&1
tail -2 gpurun_out/$1/ncu.txt
