# scratch GPU job: pipelined C4 bench (600 frames) of the in-tree build vs ab/<variants>, twice
mkdir -p gpurun_out/$1
N=$1; shift
for V in new "$@" new "$@"; do
  if [ "$V" = new ]; then timeout 600 python bench.py --steps 600 --warmup 5 --no-cpu-baseline > gpurun_out/$N/b.txt 2>&1;
  else GSC_AB_LIB=$PWD/ab/$V/libgscache.so timeout 600 python bench.py --steps 600 --warmup 5 --no-cpu-baseline > gpurun_out/$N/b.txt 2>&1; fi
  tail -1 gpurun_out/$N/b.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$V', d['value'], d['serial_ms_per_frame'], d['stages']['blend']['ms_per_frame'])"
done
