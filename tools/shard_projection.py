"""Strong-scaling PROJECTION from single-GPU shard runs (this pool gives one GPU per call; not a multi-GPU
measurement).  For N in 1, 2, 4, 8 it times, on one B200 and through the same C-ABI call bench.py uses, rank 0's shard
[0, m/N) of the config (the largest shard; all shards are within one SNP of each other) in bench.py's headline
configuration (FP64 DMMA, overlap, auto block size, X_R resident in HBM), and reports
    projected GLS/s(N) = m t / T_shard(N)          (the max over ranks is the largest shard's time)
    efficiency(N)      = GLS/s(N) / (N GLS/s(1))
The one state broadcast of setup (1.36 GB at C4 over NVLink) is outside the timed region, as in bench.py.
    python tools/shard_projection.py [--config 4] [--steps 2] > profiles/scaling_projection_r02.json
Not product code."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import datagen  # noqa: E402
import paper_1207_2169_b200 as gw  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    cfg = datagen.CONFIGS[a.config]
    dev = torch.device("cuda", 0)
    ds = datagen.dataset(cfg, device=dev)
    ld = (cfg.n + 15) // 16 * 16
    xr_h = torch.empty((cfg.m, ld), dtype=torch.uint8, pin_memory=True)
    datagen.xr_dosages(cfg, ld=ld, out=xr_h.numpy())
    xr = xr_h.to(dev)
    del xr_h
    eng = gw.Gwas(cfg.n, cfg.p, cfg.t, device=0, block_cols=0, overlap=True)
    eng.setup(ds.Phi, ds.XL, ds.Y, ds.h2, ds.s2)
    out = eng.alloc_outputs(cfg.m)
    rows = []
    for n_gpus in (1, 2, 4, 8):
        lo, hi = bench.shard_range(cfg.m, 0, n_gpus, "strong")
        o = (out[0][lo:hi], out[1][lo:hi], out[2][lo:hi])
        for _ in range(a.warmup):
            eng.run(xr[lo:hi], out=o)
        with bench.ClockSampler(bench.nvml_id(dev)) as clk:
            ms = bench._timed_steps(eng, xr[lo:hi], o, a.steps, eng.compute_stream, torch.cuda.synchronize)
        t_shard = ms / a.steps
        rows.append({"n_gpus": n_gpus, "shard_snps": hi - lo, "ms_per_step_shard": t_shard,
                     "projected_gls_per_s": cfg.m * cfg.t / (t_shard / 1e3), "clocks": clk.summary()})
    base = rows[0]["projected_gls_per_s"]
    for r in rows:
        r["projected_efficiency"] = r["projected_gls_per_s"] / (r["n_gpus"] * base)
    print(json.dumps({"what": "strong-scaling projection from single-B200 shard runs (NOT a multi-GPU measurement)",
                      "config": f"{cfg.name}: n={cfg.n}, p={cfg.p}, m={cfg.m}, t={cfg.t}",
                      "block_cols": eng.run_info()["block_cols"], "rows": rows,
                      "excluded": "the one setup broadcast of the state (bench.py reports it as setup.ms_broadcast)"}))
    eng.close()


if __name__ == "__main__":
    main()
