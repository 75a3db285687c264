# scratch GPU job: ncu launch list (gpu__time_duration) of kernels matching $2, skipping $3 launches, $4 launches, bench of $5 steps
mkdir -p gpurun_out/$1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:$2" -s ${3:-0} -c ${4:-20} --csv --log-file gpurun_out/$1/launches.csv python bench.py --steps ${5:-300} --warmup 3 --no-cpu-baseline > gpurun_out/$1/ncu.txt 2>&1
python tools/ncu_launch_summary.py gpurun_out/$1/launches.csv
