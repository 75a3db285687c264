# final sanity: smoke, default bench (no flags), reference arm, 2-rank (shared GPU) bench
mkdir -p gpurun_out/$1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/$1/bench_default.txt 2>&1; tail -1 gpurun_out/$1/bench_default.txt | cut -c1-300
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/$1/bench_ref.txt 2>&1; tail -1 gpurun_out/$1/bench_ref.txt | cut -c1-300
GSC_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/$1/bench_2rank.txt 2>&1; tail -1 gpurun_out/$1/bench_2rank.txt | cut -c1-200
