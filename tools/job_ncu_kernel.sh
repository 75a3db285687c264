# scratch GPU job: ncu --set full (with source) of one launch of the kernels matching $2 at C4 trajectory
# frame $3 (default 50), for the current build and optional ab/<variant> libraries ($4...).
#   bash tools/job_ncu_kernel.sh <outdir> <kernel regex> [frame] [variants...]
mkdir -p gpurun_out/$1
OUT=$1; RX=$2; F=${3:-50}; shift 3
cat > /tmp/one_frame_k.py <<'PY'
import os, sys
if os.environ.get("GSC_AB_LIB"):
    from paper_2502_14938_b200 import _abi
    _abi.SO_PATH = os.environ["GSC_AB_LIB"]
import torch, scenegen as sg, paper_2502_14938_b200 as gp
cfg = sg.config("C4"); traj = sg.trajectory(cfg); f = int(sys.argv[1])
r = gp.Renderer(0, cfg.width, cfg.height, cfg.fov_y_deg, cfg.near, cfg.far, cfg.d_max).load(cfg.scene())
o = r.alloc_outputs(gp.GSC_FMT_RGBA8)
for k in range(f - 12, f + 1):
    r.render_into(traj[k], *o, gp.GSC_FMT_RGBA8)
torch.cuda.synchronize()
PY
for V in cur "$@"; do
  case $V in cur) ENV="";; *) ENV="GSC_AB_LIB=$PWD/ab/$V/libgscache.so";; esac
  env $ENV PYTHONPATH=. timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$RX" -s 12 -c 1 -o gpurun_out/$OUT/k_$V python /tmp/one_frame_k.py $F > gpurun_out/$OUT/ncu_$V.txt 2>&1
  tail -1 gpurun_out/$OUT/ncu_$V.txt
done
