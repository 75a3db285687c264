# Round profile job (run from the repo root on the GPU box): tests, bench lines, sanitizer, launch list,
# ncu captures.  Outputs under gpurun_out/prof/.
set -x
mkdir -p gpurun_out/prof
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/prof/smi.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/prof/smoke.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/prof/pytest_gpu.txt 2>&1
python bench.py --steps 600 --warmup 5 > gpurun_out/prof/bench_C4.txt 2>&1
python bench.py --steps 600 --warmup 5 --no-cpu-baseline --stagger > gpurun_out/prof/bench_C4_stagger.txt 2>&1
python bench.py --config C5 --steps 600 --warmup 5 --no-cpu-baseline > gpurun_out/prof/bench_C5.txt 2>&1
python bench.py --impl reference --steps 4 --warmup 3 > gpurun_out/prof/bench_ref.txt 2>&1
GSC_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 300 --warmup 5 --no-cpu-baseline > gpurun_out/prof/bench_2rank.txt 2>&1
timeout 800 python tools/cull_scale.py 18000000 60 gpurun_out/prof/cull_18M.json > gpurun_out/prof/cull_18M.txt 2>&1
{ echo "## memcheck"; timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -q -k "c1_all or reset or rgba8 or c1_abl or dered or host_async or c1_guide or stagger" 2>&1 | tail -4; echo "memcheck_rc=$?";
  echo "## racecheck"; timeout 600 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -q -k "c1_all or stagger" 2>&1 | tail -3;
  echo "## synccheck"; timeout 600 compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_parity.py -q -k "c1_all or stagger" 2>&1 | tail -3; } > gpurun_out/prof/sanitizer.txt 2>&1
PYTHONPATH=. timeout 300 python tools/elastic_session.py C4 15 72 120 2 gpurun_out/prof/elastic_C4.json > gpurun_out/prof/elastic.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/prof/launches.csv python bench.py --steps 40 --warmup 3 --no-cpu-baseline > gpurun_out/prof/ncu_launch_run.txt 2>&1
# one mid-trajectory frame: warm-up 3 frames + 97 timed = frame ~100 of the trajectory, 17 launches per frame
ncu --set full --clock-control none --import-source on -s 1700 -c 17 -o gpurun_out/prof/frame100 python bench.py --steps 110 --warmup 3 --no-cpu-baseline > gpurun_out/prof/ncu_full_run.txt 2>&1
