# Round profile job (run from the repo root on the GPU box): bench lines, launch list, ncu captures.
set -x
mkdir -p gpurun_out/prof
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/prof/smoke.txt 2>&1
python bench.py --steps 600 --warmup 5 > gpurun_out/prof/bench_C4.txt 2>&1
python bench.py --config C5 --steps 600 --warmup 5 --no-cpu-baseline > gpurun_out/prof/bench_C5.txt 2>&1
python bench.py --impl reference --steps 4 --warmup 3 > gpurun_out/prof/bench_ref.txt 2>&1
GSC_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 300 --warmup 5 --no-cpu-baseline > gpurun_out/prof/bench_2rank.txt 2>&1
PYTHONPATH=. timeout 300 python tools/elastic_session.py C4 15 72 120 2 gpurun_out/prof/elastic_C4.json > gpurun_out/prof/elastic.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/prof/launches.csv python bench.py --steps 40 --warmup 3 --no-cpu-baseline > gpurun_out/prof/ncu_launch_run.txt 2>&1
ncu --set full --clock-control none --import-source on -s 1398 -c 14 -o gpurun_out/prof/frame100 python bench.py --steps 110 --warmup 3 --no-cpu-baseline > gpurun_out/prof/ncu_full_run.txt 2>&1
