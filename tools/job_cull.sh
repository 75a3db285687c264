# scratch GPU job: C4/C5 cull parity + timing + ncu full capture of cull_classify
mkdir -p gpurun_out/$1
timeout 500 python -m pytest tests -x -q -m gpu -k "c1_all_poses or c1_moving or c3_trajectory or c4_full or reset_and_empty or c5_full" > gpurun_out/$1/pytest_gpu.txt 2>&1
tail -2 gpurun_out/$1/pytest_gpu.txt
for C in C4 C5; do
timeout 400 python bench.py --config $C --steps 300 --warmup 5 --no-cpu-baseline > gpurun_out/$1/bench_$C.txt 2>&1
tail -1 gpurun_out/$1/bench_$C.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], {k:(v['ms_per_frame'],v['GBps']) for k,v in d['stages'].items()})"
timeout 400 ncu --set full --clock-control none --import-source on -k regex:cull_classify -s 100 -c 2 -o gpurun_out/$1/cull_$C python bench.py --config $C --steps 110 --warmup 3 --no-cpu-baseline > gpurun_out/$1/ncu_$C.txt 2>&1
done
