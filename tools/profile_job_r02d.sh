# Round-2 final refresh profile job (session 3 final: packed blend + staging prefetch, pipelined fixup, cull, emit count parking) (run from the repo root on the GPU box): tests, bench lines, sanitizer, launch list,
# ncu captures, F2 zoom-out, cull at City scale.  Outputs under gpurun_out/prof_r02/.
set -x
O=gpurun_out/prof_r02d
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv > $O/smi.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu.txt 2>&1
python bench.py --steps 600 --warmup 5 > $O/bench_C4.txt 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_C4_20.txt 2>&1
python bench.py --steps 600 --warmup 5 --no-cpu-baseline --stagger > $O/bench_C4_stagger.txt 2>&1
python bench.py --steps 600 --warmup 5 --no-cpu-baseline --blend-exact > $O/bench_C4_blend_exact.txt 2>&1
python bench.py --config C5 --steps 600 --warmup 5 --no-cpu-baseline > $O/bench_C5.txt 2>&1
python bench.py --impl reference --steps 4 --warmup 3 > $O/bench_ref.txt 2>&1
GSC_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 300 --warmup 5 --no-cpu-baseline > $O/bench_2rank.txt 2>&1
timeout 900 python tools/cull_scale.py 18000000 60 $O/cull_18M.json > $O/cull_18M.txt 2>&1
PYTHONPATH=. timeout 600 python tools/stage_profile.py C4 600 50 > $O/stage_profile_C4.txt 2>&1
# compute-sanitizer is closed on the pool: the bounds-checked debug library instead (tools/bounds_build.py, built before the job)
GSC_AB_LIB=$PWD/ab/bounds/libgscache.so timeout 2400 python -m pytest tests -q -m gpu > $O/pytest_bounds.txt 2>&1
GSC_AB_LIB=$PWD/ab/bounds/libgscache.so PYTHONPATH=. timeout 600 python tools/stage_profile.py C4 600 100 > $O/stage_bounds.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $O/launches.csv python bench.py --steps 40 --warmup 3 --no-cpu-baseline > $O/ncu_launch_run.txt 2>&1
# one mid-trajectory frame: warm-up 3 frames + reset (1 kernel) + 97 timed frames, 18 launches per frame
ncu --set full --clock-control none --import-source on -s $((3 * 18 + 1 + 97 * 18)) -c 18 -o $O/frame100 python bench.py --steps 110 --warmup 3 --no-cpu-baseline > $O/ncu_full_run.txt 2>&1
