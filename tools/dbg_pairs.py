import numpy as np, oracle, scenegen as sg, sys
sys.path.insert(0,'tests')
from parity import renderer, oracle_config
cfg=sg.config('C1'); sc=cfg.scene()
o=oracle.Oracle(sc, oracle_config(oracle,cfg)); r=renderer(cfg).load(sc)
rig=sg.trajectory(cfg)[0]
o.frame(rig); r.render(rig)
ok,og=o.pairs(); gk,gg=r.debug('pairs'),r.debug('pair_g')
d=np.nonzero(gk!=ok)[0]
print('n',len(ok),len(gk),'ndiff',len(d))
for i in d[:10]:
    print(i, hex(int(gk[i])), hex(int(ok[i])), gg[i], og[i])
print('tiles gpu', np.unique(gk>>np.uint64(32))[:20])
