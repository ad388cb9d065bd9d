"""Small run of every kernel (setup, K1/K2 FP64, int8-sliced, K3, staging, overlap) for compute-sanitizer.
Not product code.  python tools/sanitize_c0.py"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import datagen
import paper_1207_2169_b200 as gw

cfg = datagen.custom_config(n=200, p=4, m=600, t=4, index=0)
ds = datagen.dataset(cfg)
XR = torch.from_numpy(datagen.xr_dosages(cfg, ld=208))
for i8 in (0, 8):
    for ovl in (False, True):
        eng = gw.Gwas(cfg.n, cfg.p, cfg.t, block_cols=256, int8_slices=i8, overlap=ovl, output_mode="full")
        eng.setup(ds.Phi, ds.XL, ds.Y, ds.h2, ds.s2)
        eng.run(XR.cuda())
        eng.run(XR.pin_memory())
        torch.cuda.synchronize()
        eng.close()
print("sanitize run ok")
