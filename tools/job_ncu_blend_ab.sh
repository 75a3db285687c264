# scratch GPU job: ncu --set full of the blend at trajectory frame $2 for the current build (fast), the exact
# kernel (GSC_F_BLEND_EXACT) and an ab/<variant> library
mkdir -p gpurun_out/$1
F=${2:-250}
cat > /tmp/one_frame.py <<'PY'
import os, sys
if os.environ.get("GSC_AB_LIB"):
    from paper_2502_14938_b200 import _abi
    _abi.SO_PATH = os.environ["GSC_AB_LIB"]
import torch, scenegen as sg, paper_2502_14938_b200 as gp
cfg = sg.config("C4"); traj = sg.trajectory(cfg); f = int(sys.argv[1])
flags = gp.GSC_F_BLEND_EXACT if os.environ.get("EXACT") else 0
r = gp.Renderer(0, cfg.width, cfg.height, cfg.fov_y_deg, cfg.near, cfg.far, cfg.d_max, flags=flags).load(cfg.scene())
o = r.alloc_outputs(gp.GSC_FMT_RGBA8)
for k in range(f - 12, f + 1):
    r.render_into(traj[k], *o, gp.GSC_FMT_RGBA8)
torch.cuda.synchronize()
PY
for V in fast exact $3; do
  case $V in fast) ENV="";; exact) ENV="EXACT=1";; *) ENV="GSC_AB_LIB=$PWD/ab/$V/libgscache.so";; esac
  env $ENV PYTHONPATH=. timeout 600 ncu --set full --clock-control none --import-source on -k regex:"blend_kernel|blend_exact_kernel" -s 12 -c 1 -o gpurun_out/$1/blend_$V python /tmp/one_frame.py $F > gpurun_out/$1/ncu_$V.txt 2>&1
  tail -1 gpurun_out/$1/ncu_$V.txt
done
