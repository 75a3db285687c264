# scratch GPU job: ncu --set full of the blend kernel at frames ~20 and ~250 (bench C4), source-level counts
mkdir -p gpurun_out/$1
for F in ${2:-20 250}; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:blend_kernel -s $F -c 1 -o gpurun_out/$1/blend$F python bench.py --steps $((F + 10)) --warmup 3 --no-cpu-baseline > gpurun_out/$1/ncu_full$F.txt 2>&1
tail -1 gpurun_out/$1/ncu_full$F.txt
done
