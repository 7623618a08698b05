import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from vi_synth import CONFIGS, make_weights, make_features
import gpu_harness as Hh
cfg = CONFIGS["C3S"].replace(t_new=3)
w = make_weights(cfg, seed=1, variant="sensitive")
g = Hh.GpuStream(cfg, w)
fid = 0
for n in [3, 1, 2, 3, 1]:
    print("push", n, "state before", g.ctx.state()[2], flush=True)
    feats = make_features(cfg, n, first_frame=fid, seed=0); fid += n
    g.step(feats)
    print("ok", flush=True)
