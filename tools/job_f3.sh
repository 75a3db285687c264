# F3 depth-policy study on the GPU: accelerating (C3A) and staged (C3T) head turns, the three guiding functions
# and staggered expiry against the uncached reference; per-frame depth / update-rate / PSNR traces
mkdir -p gpurun_out/f3
for C in C3A C3T; do
  PYTHONPATH=. timeout 1200 python tools/quality.py $C 300 gpurun_out/f3/quality_$C.json method,guide_exponential,guide_staged,stagger,no_reuse > gpurun_out/f3/quality_$C.txt 2>&1
  tail -5 gpurun_out/f3/quality_$C.txt
done
