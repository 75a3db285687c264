# scratch GPU job: A/B stage profile (C4, 300 frames, buckets of 100) of the in-tree build vs ab/<variants>, twice
mkdir -p gpurun_out/$1
N=$1; shift
for V in new "$@" new "$@"; do
  echo "== $V"
  if [ "$V" = new ]; then PYTHONPATH=. timeout 300 python tools/stage_profile.py C4 300 100;
  else GSC_AB_LIB=$PWD/ab/$V/libgscache.so PYTHONPATH=. timeout 300 python tools/stage_profile.py C4 300 100; fi
done > gpurun_out/$N/ab.txt 2>&1
grep -vE "^frames" gpurun_out/$N/ab.txt
