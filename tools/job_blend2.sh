# scratch GPU job: packed blend -- smoke, GPU tests, A/B stage profile against ab/$2 variants, C4 bench
mkdir -p gpurun_out/$1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$1/smoke.txt 2>&1; tail -1 gpurun_out/$1/smoke.txt
timeout 1500 python -m pytest tests -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/$1/pytest_gpu.txt 2>&1
tail -3 gpurun_out/$1/pytest_gpu.txt
for V in new $2 new $2; do
  echo "== $V"
  if [ "$V" = new ]; then PYTHONPATH=. timeout 300 python tools/stage_profile.py C4 300 100;
  else GSC_AB_LIB=$PWD/ab/$V/libgscache.so PYTHONPATH=. timeout 300 python tools/stage_profile.py C4 300 100; fi
done > gpurun_out/$1/ab.txt 2>&1
grep -E "==|blend|total" gpurun_out/$1/ab.txt | head -40
timeout 400 python bench.py --steps 300 --warmup 5 --no-cpu-baseline > gpurun_out/$1/bench_C4.txt 2>&1
tail -1 gpurun_out/$1/bench_C4.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['serial_ms_per_frame'], d['frame_counts']['blend_fixup_pixels']); print({k:v['ms_per_frame'] for k,v in d['stages'].items()})"
