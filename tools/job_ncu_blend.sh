# scratch GPU job: failed GPU tests rerun + ncu --set full of one mid-trajectory blend launch (frame ~100)
mkdir -p gpurun_out/$1
timeout 1500 python -m pytest tests -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/$1/pytest_gpu.txt 2>&1
tail -3 gpurun_out/$1/pytest_gpu.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:blend_kernel -s 100 -c 1 -o gpurun_out/$1/blend100 python bench.py --steps 110 --warmup 3 --no-cpu-baseline > gpurun_out/$1/ncu_full.txt 2>&1
tail -2 gpurun_out/$1/ncu_full.txt
