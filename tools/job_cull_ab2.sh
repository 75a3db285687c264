# scratch GPU job: cull at 18M anchors (cold L2), in-tree build vs ab/<variants>
mkdir -p gpurun_out/$1
N=$1; shift
for V in new "$@" new "$@"; do
  if [ "$V" = new ]; then timeout 600 python tools/cull_scale.py 18000000 30 > gpurun_out/$N/c.txt 2>&1;
  else GSC_AB_LIB=$PWD/ab/$V/libgscache.so timeout 600 python tools/cull_scale.py 18000000 30 > gpurun_out/$N/c.txt 2>&1; fi
  echo "$V $(tail -1 gpurun_out/$N/c.txt | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_frame"], d["frac"])')"
done
