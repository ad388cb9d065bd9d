"""One block of K1 -> K2 -> K3 at a config's full n, p, t (for ncu captures).  Not product code.
    python tools/profile_kernels.py --config 4 [--cols 8192] [--reps 1]"""
import argparse, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import datagen
import paper_1207_2169_b200 as gw

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--cols", type=int, default=8192)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--int8-slices", type=int, default=0)
ap.add_argument("--n", type=int, default=None, help="override n (config-0 generators at that size)")
ap.add_argument("--t", type=int, default=None)
ap.add_argument("--trait-rank", type=int, default=0)
a = ap.parse_args()
cfg = datagen.CONFIGS[a.config]
if a.n or a.t:
    cfg = datagen.custom_config(n=a.n or cfg.n, p=cfg.p, m=max(a.cols, 1), t=a.t or cfg.t, S=2 * (a.n or cfg.n), index=500)
ld = (cfg.n + 15) // 16 * 16
ds = datagen.dataset(cfg, device="cuda")
XR = torch.from_numpy(datagen.xr_dosages(cfg, 0, a.cols, ld=ld)).cuda()
eng = gw.Gwas(cfg.n, cfg.p, cfg.t, block_cols=a.cols, timing=True, int8_slices=a.int8_slices,
              trait_rank=a.trait_rank)
eng.setup(ds.Phi, ds.XL, ds.Y, ds.h2, ds.s2)
out = eng.alloc_outputs(a.cols)
for _ in range(a.reps):
    eng.run(XR, out=out)
torch.cuda.synchronize()
kt = eng.kernel_times()
print("trait rank", eng.trait_rank(), eng.timings())
print(f"n={cfg.n} t={cfg.t} cols={a.cols}", {k: round(v['ms'] / max(1, v['launches']), 4) for k, v in kt.items()})
