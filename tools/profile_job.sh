set -x
mkdir -p gpurun_out/p60
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/p60/smoke.txt 2>&1
python bench.py --steps 600 --warmup 5 > gpurun_out/p60/bench_C4.txt 2>&1
python bench.py --config C5 --steps 600 --warmup 5 --no-cpu-baseline > gpurun_out/p60/bench_C5.txt 2>&1
python bench.py --impl reference --steps 4 --warmup 3 > gpurun_out/p60/bench_ref.txt 2>&1
GSC_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 300 --warmup 5 --no-cpu-baseline > gpurun_out/p60/bench_2rank.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/p60/launches.csv python bench.py --steps 40 --warmup 3 --no-cpu-baseline > gpurun_out/p60/ncu_launch_run.txt 2>&1
ncu --set full --clock-control none --import-source on -s 1400 -c 14 -o gpurun_out/p60/frame100 python bench.py --steps 110 --warmup 3 --no-cpu-baseline > gpurun_out/p60/ncu_full_run.txt 2>&1
