# scratch GPU job: ncu --set full of derive_mma on a flush frame (trajectory frame 10) and a steady frame (15)
mkdir -p gpurun_out/$1
cat > /tmp/derive_frames.py <<'PY'
import torch, scenegen as sg, paper_2502_14938_b200 as gp
cfg = sg.config("C4"); traj = sg.trajectory(cfg)
r = gp.Renderer(0, cfg.width, cfg.height, cfg.fov_y_deg, cfg.near, cfg.far, cfg.d_max).load(cfg.scene())
o = r.alloc_outputs(gp.GSC_FMT_RGBA8)
for k in range(16):
    r.render_into(traj[k], *o, gp.GSC_FMT_RGBA8)
torch.cuda.synchronize()
print([h["n_misses"] for h in r.stats_history(16)])
PY
PYTHONPATH=. timeout 600 ncu --set full --clock-control none --import-source on -k regex:derive_mma ${NCU_EXTRA} -o gpurun_out/$1/derive python /tmp/derive_frames.py > gpurun_out/$1/ncu_derive.txt 2>&1
tail -3 gpurun_out/$1/ncu_derive.txt
