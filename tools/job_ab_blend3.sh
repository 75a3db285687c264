# scratch GPU job: GPU parity subset, then A/B stage profile (C4, 300 frames) of the in-tree build vs ab/<variants>
mkdir -p gpurun_out/$1
N=$1; shift
timeout 900 python -m pytest tests -x -q -m gpu -k "c1_all_poses or c1_moving or c3_trajectory or c4_full or fast_exp or ragged or c1_abl" > gpurun_out/$N/pytest_gpu.txt 2>&1
tail -2 gpurun_out/$N/pytest_gpu.txt
for V in new "$@" new "$@"; do
  echo "== $V"
  if [ "$V" = new ]; then PYTHONPATH=. timeout 300 python tools/stage_profile.py C4 300 100;
  else GSC_AB_LIB=$PWD/ab/$V/libgscache.so PYTHONPATH=. timeout 300 python tools/stage_profile.py C4 300 100; fi
done > gpurun_out/$N/ab.txt 2>&1
python - gpurun_out/$N/ab.txt <<'PY'
import sys
cur=None
for l in open(sys.argv[1]):
    if l.startswith('=='): cur=l.split()[1]; out=[]
    elif l.strip() and l.split()[0][0].isdigit():
        f=l.split(); print(cur, f[0]+f[1] if f[1][0]=='-' else f[0], 'blend', f[-5] if len(f)>12 else f[8], 'total', f[-4] if len(f)>12 else f[9])
PY
