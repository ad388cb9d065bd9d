"""Small run of every kernel and of the three-stream pipeline for compute-sanitizer (racecheck / synccheck /
memcheck): setup, K1/K2 FP64 (fused and unfused), int8-sliced, K3, host staging on the copy stream, the overlap
(auxiliary) stream, host outputs on the D2H stream, and back-to-back gwas_run calls into different buffers.
Not product code.  python tools/sanitize_c0.py"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import datagen
import paper_1207_2169_b200 as gw

for t in (4, 12):   # t = 4: K2 fused into K1 (t (p+2) = 24 <= 28); t = 12: separate K2 product
    cfg = datagen.custom_config(n=200, p=4, m=600, t=t, index=0)
    ds = datagen.dataset(cfg)
    XR = torch.from_numpy(datagen.xr_dosages(cfg, ld=208))
    xr_h, xr_d = XR.pin_memory(), XR.cuda()
    for i8 in (0, 8):
        for ovl in (False, True):
            eng = gw.Gwas(cfg.n, cfg.p, cfg.t, block_cols=256, int8_slices=i8, overlap=ovl, output_mode="full")
            eng.setup(ds.Phi, ds.XL, ds.Y, ds.h2, ds.s2)
            ref = [x.clone() for x in eng.run(xr_d)]
            outs = [eng.alloc_outputs(cfg.m, host=h) for h in (False, True, True)]
            eng.run(xr_h, out=outs[0])
            eng.run(xr_h, out=outs[1])        # back to back: staging buffers and host-output sets reused
            eng.run(xr_d, out=outs[2])
            torch.cuda.synchronize()
            for o in outs:
                for a, b in zip(ref, o):
                    assert torch.equal(a.cpu(), b.cpu())
            eng.close()
print("sanitize run ok")
