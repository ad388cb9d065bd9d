#!/usr/bin/env python
"""Benchmark of the B200-native CLAK-Eig GLS-sequence hot path (BASELINE.json metric: GLS/s = SNP x trait pairs
per second, with the FP64 tensor-pipe fraction of peak).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...          (one process per GPU, NCCL)

A step = one pass of the whole hot path (Alg. 4 line 3 + lines 13-16: K1 rotation
GEMM, K2 weighted-reduction GEMM, K3 Schur solve) over every SNP of the rank's shard, for all t traits.
Setup (dsyevd, precompute, the one NCCL broadcast of the replicated state) is timed and reported separately.
Scaling is weak: every rank processes its own m SNPs of the config (rank r takes SNP columns [r m, (r+1) m) of
an N*m-SNP synthetic genome), so `value` = N*m*t / (max over ranks of the step time).

`value`: X_R already resident in HBM (uint8 dosages, exact), K1/K2 on the FP64 DMMA pipe (the north star's
         design), blocks pipelined over two streams; timed with CUDA events on the compute stream.
`roofline`: K1 from a serial pass of the same run (per-launch CUDA events; overlapped launches would share SMs).
`modes.int8_sliced`: the exact int8-sliced tcgen05 mode on the same inputs.
`e2e`:   the same through the public API from pinned HOST X_R (block staging on the copy stream inside the timed
         region) plus the device->host read of every step's b, Var and status.
`--impl reference`: the CPU oracle (oracle/), as it stands, on a bounded sample of the same workload (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import datagen  # noqa: E402

METRIC = "GLS/s (SNP x trait pairs)"
UNIT = "GLS/s"


# ------------------------------------------------------------------ host-side helpers (CPU-testable)
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def shard_range(m: int, rank: int, world: int, scaling: str = "weak"):
    """SNP columns of a rank.  weak: [rank*m, (rank+1)*m) of an N*m genome; strong: contiguous split of m."""
    if scaling == "weak":
        return rank * m, (rank + 1) * m
    return (rank * m) // world, ((rank + 1) * m) // world


def max_over_ranks(x: float, world: int, device=None) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replicate_state(state, world: int, src: int = 0):
    """Alg. 4's per-trait precomputation is done once on rank `src`; every other rank receives the state bytes
    (Z, W, B_op/D, per-trait factors) through ONE broadcast -- the only collective of the method."""
    if world > 1:
        import torch.distributed as dist
        dist.broadcast(state, src=src)
    return state


def flops_per_block(n, p, t, cols):
    """Algorithmic flops: K1 2 n^2 k, K2 2 n k t (p+2); K3 ~ k t (p^2 + 4p + 8)."""
    return {"K1": 2.0 * n * n * cols, "K2": 2.0 * n * cols * t * (p + 2), "K3": cols * t * (p * p + 4 * p + 8.0)}


def k3_bytes(p, t, cols, full=False):
    """K3 algorithmic HBM bytes: reads 8 (p+2) per pair, writes 8+8+1 (SNP mode) or 16 (p+1)+1 (full)."""
    w = p + 1
    return cols * t * (8 * (p + 2) + (16 * w + 1 if full else 17))


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms while the timed region runs."""
    FIELDS = "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._th = None

    def _loop(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5).stdout
                vals = [v.strip() for v in out.strip().split(",")]
                if len(vals) >= 8:
                    self.rows.append(vals)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._th = threading.Thread(target=self._loop, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._th:
            self._th.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        smax = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(self.rows),
                "power_w_max": max((float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()), default=None)}


def fp64_peak():
    """Measured FP64 DMMA peak (tools/fp64_peak.cu on this pool's B200: back-to-back mma.sync.m8n8k4.f64 on all
    SMs, profiles/fp64_peak_r01.json).  MEASURED_PEAKS.json has no FP64 entry."""
    path = os.path.join(ROOT, "profiles", "fp64_peak_r01.json")
    with open(path) as f:
        d = json.load(f)
    return float(d["dmma_tflops"]), "measured: tools/fp64_peak.cu DMMA.8x8x4 microbenchmark (profiles/fp64_peak_r01.json)"


def ncu_traffic():
    path = os.path.join(ROOT, "profiles", "k1_traffic.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f)
    return None


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


# ------------------------------------------------------------------ oracle (cpu_baseline / --impl reference)
def oracle_sample(cfg, ds, traits, snps):
    """Time the CPU oracle, as it stands, on (snps x traits) of the config.  Returns (pairs, seconds, threads)."""
    import scipy.linalg  # noqa: F401  (loads the LAPACK the oracle uses)
    import threadpoolctl

    import oracle
    G = datagen.xr_columns(cfg, snps)
    t0 = time.perf_counter()
    oracle.gls_sequence(ds.Phi, ds.XL, G, ds.Y, ds.h2, ds.s2, traits=traits)
    dt = time.perf_counter() - t0
    info = threadpoolctl.threadpool_info()
    threads = max([i.get("num_threads", 1) for i in info] or [1])
    return len(snps) * len(traits), dt, threads


# ------------------------------------------------------------------ our arm
def _timed_steps(eng, xr, out, steps, stream, barrier):
    """`steps` full passes of the hot path between a barrier + synchronize on both sides; CUDA events on the
    compute stream.  Returns ms."""
    import torch
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        eng.run(xr, out=out)
    e1.record(stream)
    barrier()
    return e0.elapsed_time(e1)


def _kernel_pass(eng, xr, out, steps, barrier):
    """Serial (non-overlapped) passes with per-launch CUDA events: the per-kernel durations behind `roofline`."""
    eng.run(xr, out=out)
    barrier()
    eng.kernel_times(reset=True)
    for _ in range(steps):
        eng.run(xr, out=out)
    barrier()
    return eng.kernel_times(reset=True)


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    # GWAS_BENCH_BACKEND=gloo (testing only): exercise the multi-rank path (broadcast + attach, max over ranks) with
    # all ranks on the visible GPU(s); NCCL needs one GPU per rank.  Numbers from such a run are not bench values.
    backend = os.environ.get("GWAS_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    import paper_1207_2169_b200 as gw

    cfg = datagen.CONFIGS[args.config]
    m_rank = cfg.m if args.snps is None else args.snps
    lo, hi = shard_range(m_rank, rank, world, args.scaling)
    if args.scaling == "weak":
        gcfg = datagen.Config(cfg.index, cfg.n, cfg.p, m_rank * world, cfg.t, cfg.S, cfg.h2_range, cfg.s2_range)
    else:
        gcfg = datagen.Config(cfg.index, cfg.n, cfg.p, m_rank, cfg.t, cfg.S, cfg.h2_range, cfg.s2_range)
    ncols = hi - lo
    n, p, t = cfg.n, cfg.p, cfg.t
    ld = (n + 15) // 16 * 16

    # inputs: the replicated part on every rank (deterministic), X_R shard in pinned host memory
    t0 = time.perf_counter()
    ds = datagen.dataset(cfg, device=dev)
    xr_host = torch.empty((ncols, ld), dtype=torch.uint8, pin_memory=True)
    datagen.xr_dosages(gcfg, lo, hi, ld=ld, out=xr_host.numpy())
    t_gen = time.perf_counter() - t0

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()

    def make_engine(i8, overlap, algorithm="eig", trait_rank=0):
        """Rank 0 sets up (eig + precompute), the state is replicated by ONE broadcast, other ranks attach."""
        eng = gw.Gwas(n, p, t, device=local, block_cols=args.block, timing=True, int8_slices=i8, overlap=overlap,
                      algorithm=algorithm, fuse_k2=bool(args.fuse_k2), trait_rank=trait_rank)
        info = {}
        if rank == 0:
            eng.setup(ds.Phi, ds.XL, ds.Y, ds.h2, ds.s2)
            info.update(eng.timings())
        if world > 1:
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            replicate_state(eng.state, world)   # the one collective: replicated setup state over NVLink
            e1.record()
            barrier()
            info["ms_broadcast"] = e0.elapsed_time(e1)
            info["broadcast_bytes"] = eng.state_bytes
            if rank != 0:
                eng.attach()
        # a second, serial context on the same state (gwas_attach) times the kernels one by one
        ser = gw.Gwas(n, p, t, device=local, block_cols=args.block, timing=True, int8_slices=i8, overlap=False,
                      algorithm=algorithm, fuse_k2=bool(args.fuse_k2), trait_rank=trait_rank)
        ser.state.copy_(eng.state)
        ser.attach()
        return eng, ser, info

    xr_dev = xr_host.to(dev)
    out = None
    blocks = [min(args.block, ncols - c) for c in range(0, ncols, args.block)]
    pairs_total = float(ncols) * t * world if args.scaling == "weak" else float(m_rank) * t
    peak, peak_src = fp64_peak()
    fl = [flops_per_block(n, p, t, c) for c in blocks]
    k1_flops = sum(f["K1"] for f in fl)
    k2_flops = sum(f["K2"] for f in fl)

    # ================= headline mode: FP64 DMMA (the north star's K1/K2) =================
    eng, ser, setup = make_engine(0, bool(args.overlap))
    out = eng.alloc_outputs(ncols)
    stream = eng.compute_stream
    for _ in range(args.warmup):
        eng.run(xr_dev, out=out)
    with ClockSampler(local) as clk:
        ms = _timed_steps(eng, xr_dev, out, args.steps, stream, barrier)
    ms_max = max_over_ranks(ms, world, dev)
    value = pairs_total * args.steps / (ms_max / 1e3)
    kt = _kernel_pass(ser, xr_dev, out, args.kernel_steps, barrier)
    k1_ms, k2_ms, k3_ms = (kt[k]["ms"] / args.kernel_steps for k in ("K1", "K2", "K3"))
    k1_tf = k1_flops / (k1_ms / 1e3) / 1e12
    k2_tf = k2_flops / (k2_ms / 1e3) / 1e12
    gemm_tf = (k1_flops + k2_flops) / ((k1_ms + k2_ms) / 1e3) / 1e12
    k3_gbs = sum(k3_bytes(p, t, c) for c in blocks) / (k3_ms / 1e3) / 1e9
    serial_ms = k1_ms + k2_ms + k3_ms

    # e2e through the public API: pinned host X_R in, pinned host (b, var, status) out -- the library stages
    # blocks H2D and streams each block's results D2H while later blocks compute
    b_h, v_h, s_h = eng.alloc_outputs(ncols, host=True)

    def e2e_step():
        eng.run(xr_host, out=(b_h, v_h, s_h))

    e2e_steps = max(1, args.e2e_steps)
    e2e_step()
    barrier()
    eng.kernel_times(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        e2e_step()
    e1.record(stream)
    barrier()
    ms_e2e = max_over_ranks(e0.elapsed_time(e1), world, dev)
    e2e_value = pairs_total * e2e_steps / (ms_e2e / 1e3)
    h2d = ((ncols - 1) * ld + n) if ncols else 0  # uint8 dosages copied per step
    kt_e2e = eng.kernel_times(reset=True)  # H2D: CUDA events around every staging copy (copy stream)
    staging_gbs = h2d * e2e_steps / (kt_e2e["H2D"]["ms"] / 1e3) / 1e9 if kt_e2e["H2D"]["ms"] > 0 else None
    d2h = b_h.numel() * 8 + v_h.numel() * 8 + s_h.numel()
    res_fp64 = (b_h.numpy().copy(), v_h.numpy().copy(), s_h.numpy().copy()) if args.check and rank == 0 else None
    eng.close()
    ser.close()
    del eng, ser

    # ================= int8-sliced mode, same inputs =================
    alt = None
    if args.int8_alt:
        S = args.int8_slices
        eng8, ser8, setup8 = make_engine(S, True)
        for _ in range(args.warmup):
            eng8.run(xr_dev, out=out)
        ms8 = max_over_ranks(_timed_steps(eng8, xr_dev, out, args.steps, eng8.compute_stream, barrier), world, dev)
        value8 = pairs_total * args.steps / (ms8 / 1e3)
        kt8 = _kernel_pass(ser8, xr_dev, out, args.kernel_steps, barrier)
        i1_ms, i2_ms, i3_ms = (kt8[k]["ms"] / args.kernel_steps for k in ("K1", "K2", "K3"))
        na_pad = (n + 63) // 64 * 64
        nlin_pad = (t * (p + 1) + 63) // 64 * 64
        i8_ops = sum(2.0 * c * (na_pad + nlin_pad) * S * n for c in blocks)   # int8 MACs x 2 actually issued
        i8_peak = 2.0 * 1623.7  # MEASURED_PEAKS bf16 x the nominal int8/bf16 ratio (4.5 / 2.25)
        k2b_flops = sum(2.0 * n * c * t for c in blocks)
        alt = {"value": value8, "unit": UNIT, "ms_per_step": ms8 / args.steps,
               "int8_slices": S,
               "representation_error": f"<= 2^-{7 * S + 1} of each digitised column's largest entry",
               "roofline": {"bound": "tensor", "kernel": f"K1i+K2a int8-sliced tcgen05 ({S} digits, TMEM int32)",
                            "achieved": i8_ops / (i1_ms / 1e3) / 1e12, "peak": i8_peak, "unit": "TOPS",
                            "frac": i8_ops / (i1_ms / 1e3) / 1e12 / i8_peak,
                            "peak_source": "MEASURED_PEAKS.json bf16_tflops x 2 (nominal int8/bf16 ratio)",
                            "fp64_equiv_tflops": (k1_flops + sum(2.0 * n * c * t * (p + 1) for c in blocks))
                                                 / (i1_ms / 1e3) / 1e12},
               "k2b_dmma_tflops": k2b_flops / (i2_ms / 1e3) / 1e12,
               "k2b_frac_of_fp64_peak": k2b_flops / (i2_ms / 1e3) / 1e12 / peak,
               "share_of_serial_step": {k: v / (i1_ms + i2_ms + i3_ms) for k, v in
                                        (("K1i+K2a", i1_ms), ("K2b", i2_ms), ("K3", i3_ms))},
               "setup": setup8}
        if args.check and rank == 0:
            torch.cuda.synchronize(dev)
            alt_res = (out[0].cpu().numpy(), out[1].cpu().numpy(), out[2].cpu().numpy())
        eng8.close()
        ser8.close()

    # ================= CLAK-Chol single-trait path (Alg. 3, NEXT-1), t == 1 only =================
    chol_modes, chol_res = {}, []
    if t == 1 and args.chol_alt:
        for i8 in (0, args.int8_slices):
            engc, serc, setupc = make_engine(i8, True, "chol")
            for _ in range(args.warmup):
                engc.run(xr_dev, out=out)
            msc = max_over_ranks(_timed_steps(engc, xr_dev, out, args.steps, engc.compute_stream, barrier), world,
                                 dev)
            ktc = _kernel_pass(serc, xr_dev, out, args.kernel_steps, barrier)
            c1_ms = ktc["K1"]["ms"] / args.kernel_steps
            tri_flops = sum(1.0 * n * n * c for c in blocks)   # L^-1 X_R: n^2 k (half of 2 n^2 k)
            entry = {"value": pairs_total * args.steps / (msc / 1e3), "unit": UNIT, "ms_per_step": msc / args.steps,
                     "K1_ms_per_step": c1_ms, "setup": setupc,
                     "K1_tflops_algorithmic": tri_flops / (c1_ms / 1e3) / 1e12}
            if i8 == 0:
                entry["K1_frac_of_fp64_peak"] = entry["K1_tflops_algorithmic"] / peak
            chol_modes["chol_int8_sliced" if i8 else "chol_fp64"] = entry
            if args.check and rank == 0:
                torch.cuda.synchronize(dev)
                chol_res.append((out[0].cpu().numpy(), out[1].cpu().numpy(), out[2].cpu().numpy()))
            engc.close()
            serc.close()

    # ================= low-rank trait weights (reading L1), FP64 and int8-sliced, many traits =================
    lr_modes, lr_res = {}, []
    if t >= 16 and args.lowrank_alt:
        for i8 in (0, args.int8_slices):
            engl, serl, setupl = make_engine(i8, True, "eig", trait_rank=-1)
            rk = engl.trait_rank() if rank == 0 else (None, None, None)
            for _ in range(args.warmup):
                engl.run(xr_dev, out=out)
            msl = max_over_ranks(_timed_steps(engl, xr_dev, out, args.steps, engl.compute_stream, barrier), world,
                                 dev)
            ktl = _kernel_pass(serl, xr_dev, out, args.kernel_steps, barrier)
            kms = {k: ktl[k]["ms"] / args.kernel_steps for k in ("K1", "K2", "K3")}
            tot = sum(kms.values())
            lr_modes["lowrank_int8_sliced" if i8 else "lowrank_fp64"] = {
                "value": pairs_total * args.steps / (msl / 1e3), "unit": UNIT, "ms_per_step": msl / args.steps,
                "trait_rank": rk[0], "sigma_ratio_dropped": (rk[2] / rk[1]) if rk[1] else None,
                "share_of_serial_step": {k: v / tot for k, v in kms.items()},
                "K2_note": "K2 = products against U_r (p r + t + r columns) + the K = r recombination", "setup": setupl}
            if args.check and rank == 0:
                torch.cuda.synchronize(dev)
                lr_res.append((out[0].cpu().numpy(), out[1].cpu().numpy(), out[2].cpu().numpy()))
            engl.close()
            serl.close()

    # ================= variance-component estimation (the paper's first step, NEXT-3) =================
    est_mode = None
    if args.est_alt and rank == 0:
        est_mode = bench_estimate(gw, cfg, ds, local, args)

    # ---------------- parity spot check on this run's outputs (outside timed regions)
    parity = None
    if args.check and rank == 0:
        parity = spot_check(cfg, gcfg, ds, lo, hi,
                            [res_fp64] + ([alt_res] if alt is not None else []) + chol_res + lr_res, args.check)
        extra = parity.pop("extra")
        if alt is not None:
            alt["parity"] = extra.pop(0)
        for name, pr in zip(list(chol_modes) + list(lr_modes), extra):
            (chol_modes if name in chol_modes else lr_modes)[name]["parity"] = pr

    res = None
    if rank == 0:
        clocks = clk.summary()
        traffic = ncu_traffic()
        res = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic (datagen, seeded)",
            "config": {"workload": f"{cfg.name}: n={n}, p={p}, m={m_rank}/rank, t={t}, k={args.block}, "
                                   f"X_R uint8 dosages resident in HBM, K1/K2 FP64 DMMA",
                       "n": n, "p": p, "m_per_rank": ncols, "t": t, "block_cols": args.block,
                       "pairs_per_step": pairs_total, "parallelism": f"snp-shard x{world}",
                       "overlap": bool(args.overlap),
                       "l2": "inputs larger than L2 (Z 0.8 GB, X_R 10 GB at C4); no flush"},
            "roofline": {"bound": "tensor", "kernel": "K1 rotation GEMM (FP64 DMMA)", "achieved": k1_tf,
                         "peak": peak, "unit": "TFLOP/s", "frac": k1_tf / peak,
                         "traffic": (traffic or {}).get("bytes_per_launch"),
                         "algorithmic_flops_per_launch": 2.0 * n * n * args.block,
                         "avg_launch_ms": kt["K1"]["ms"] / max(1, kt["K1"]["launches"]),
                         "timing": "CUDA events around every K1 launch, serial pass of the same run",
                         "peak_source": peak_src},
            "gemm_stages": {"K1_tflops": k1_tf, "K2_tflops": k2_tf, "K1K2_tflops": gemm_tf,
                            "K1K2_frac_of_peak": gemm_tf / peak, "K3_hbm_gbs": k3_gbs,
                            "share_of_serial_step": {"K1": k1_ms / serial_ms, "K2": k2_ms / serial_ms,
                                                     "K3": k3_ms / serial_ms}},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "steps": e2e_steps, "ms_per_step": ms_e2e / e2e_steps,
                    "staging_h2d_gbs": staging_gbs,
                    "staging_note": "pinned host -> HBM block copies on the copy stream (PCIe), timed by CUDA events "
                                    "around each copy while compute runs"},
            "gpu_launches": 3 * len(blocks) * args.steps,
            "setup": {**setup, "datagen_s": t_gen},
            "clocks": clocks,
        }
        if alt is not None or chol_modes or est_mode or lr_modes:
            res["modes"] = ({"int8_sliced": alt} if alt is not None else {})
            res["modes"].update(chol_modes)
            res["modes"].update(lr_modes)
            if est_mode:
                res["modes"]["estimate"] = est_mode
        if parity is not None:
            res["parity"] = parity
        if not args.no_cpu_baseline:
            pairs, sec, thr = cpu_baseline_sample(cfg, ds, args)
            res["cpu_baseline"] = {"value": pairs / sec, "unit": UNIT, "cores": thr, "kind": "oracle",
                                   "sample": f"{pairs} pairs of {cfg.name} ({args.cpu_traits} traits x "
                                             f"{args.cpu_snps} SNPs, Alg. 1 per problem, fp64 numpy/LAPACK), "
                                             f"{sec:.1f} s on {host_cores()} host cores",
                                   "projected_full_config_s": cfg.m * cfg.t / (pairs / sec)}
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return res


def est_passes(p):
    """Streaming passes over (W, X_L', y'_j) per trait in est_traits (estimate.cuh): 26 grid passes (4 grid points
    each), 2 per derivative evaluation (1 at the grid argmax + EST_ITERS bisection steps) and 2 for the final
    evaluation."""
    return 26 + 2 * (1 + 50) + 2


def bench_estimate(gw, cfg, ds, local, args):
    """gwas_setup_estimate on the config's traits (REML and ML): kernel time from CUDA events (gwas_estimate_ms),
    traits/s, the bytes the kernels stream per trait (mostly L2 hits: X_L' and W are shared by all traits), and the
    estimates against the simulated truth (reading A13).  Parity with the oracle is in tests/test_gpu_estimate.py."""
    import torch
    out = {}
    for method in ("reml", "ml"):
        eng = gw.Gwas(cfg.n, cfg.p, cfg.t, device=local, block_cols=args.block)
        ms = []
        for _ in range(2):
            est = eng.setup_estimate(ds.Phi, ds.XL, ds.Y, method)
            ms.append(eng.estimate_ms())
        tm = eng.timings()
        eng.close()
        torch.cuda.synchronize()
        k = min(ms)
        streamed = est_passes(cfg.p) * (cfg.p + 2) * 8.0 * cfg.n * cfg.t
        err = est["h2"] - ds.h2
        out[method] = {"ms": k, "traits_per_s": cfg.t / (k / 1e3), "ms_eig": tm["ms_eig"],
                       "frac_of_eig": k / tm["ms_eig"],
                       "streamed_gb_per_s": streamed / (k / 1e3) / 1e9,
                       "h2_mean_err_vs_truth": float(np.mean(err)), "h2_rmse_vs_truth": float(np.sqrt(np.mean(err ** 2))),
                       "h2_corr_vs_truth": float(np.corrcoef(est["h2"], ds.h2)[0, 1]) if cfg.t > 2 else None,
                       "sigma2_mean_ratio_vs_truth": float(np.mean(est["sigma2"] / ds.s2))}
    return out


def cpu_baseline_sample(cfg, ds, args):
    rng = np.random.default_rng(cfg.seed)
    traits = np.sort(rng.choice(cfg.t, size=min(cfg.t, args.cpu_traits), replace=False))
    snps = np.sort(rng.choice(cfg.m, size=min(cfg.m, args.cpu_snps), replace=False))
    return oracle_sample(cfg, ds, traits, snps)


def spot_check(cfg, gcfg, ds, lo, hi, results, npairs):
    """Oracle on a seeded sample of this rank's pairs (after the timed regions); `results` is a list of
    (b, var, status) host arrays from different modes, all checked against the same oracle values."""
    import oracle
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from gpu_helpers import compare
    rng = np.random.default_rng(cfg.seed + 1)
    nt = min(cfg.t, 4)
    traits = np.sort(rng.choice(cfg.t, size=nt, replace=False))
    ns = max(1, npairs // nt)
    loc = np.unique(np.concatenate([[0, hi - lo - 1], rng.choice(hi - lo, size=min(ns, hi - lo), replace=False)]))
    G = datagen.xr_columns(gcfg, loc + lo)
    ref = oracle.gls_sequence(ds.Phi, ds.XL, G, ds.Y, ds.h2, ds.s2, traits=traits)
    outs = []
    for b, v, s in results:
        eb, ev = compare(b[np.ix_(loc, traits)], v[np.ix_(loc, traits)], s[np.ix_(loc, traits)], ref)
        outs.append({"pairs": int(loc.size * nt), "max_db_over_se": eb, "max_var_rel": ev, "tol": 1e-8,
                     "pass": bool(eb <= 1e-8 and ev <= 1e-8)})
    res = dict(outs[0])
    res["extra"] = outs[1:]
    return res


# ------------------------------------------------------------------ reference arm (the oracle)
def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return None
    cfg = datagen.CONFIGS[args.config]
    dev = None
    try:
        import torch
        if torch.cuda.is_available():
            dev = torch.device("cuda", local)
    except Exception:
        pass
    ds = datagen.dataset(cfg, device=dev)
    rng = np.random.default_rng(cfg.seed + 7)
    times, pairs_all, thr = [], 0, 1
    for step in range(args.warmup + args.steps):
        traits = np.array([int(rng.integers(cfg.t))])
        snps = np.sort(rng.choice(cfg.m, size=min(cfg.m, args.ref_snps), replace=False))
        pairs, sec, thr = oracle_sample(cfg, ds, traits, snps)
        if step >= args.warmup:
            times.append(sec)
            pairs_all += pairs
    total = sum(times)
    value = pairs_all / total
    return {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic (datagen, seeded)",
            "impl": "reference",
            "config": {"workload": f"{cfg.name}: n={cfg.n}, p={cfg.p}, m={cfg.m}, t={cfg.t} -- per step a bounded "
                                   f"sample: 1 trait x {args.ref_snps} SNPs", "n": cfg.n, "p": cfg.p, "t": cfg.t},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": thr, "kind": "oracle",
                             "sample": f"per step 1 trait x {args.ref_snps} SNPs of {cfg.name}; "
                                       f"{host_cores()} host cores"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4, help="BASELINE.json config index (default 4)")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak")
    ap.add_argument("--block", type=int, default=8192, help="SNP columns per streamed block (k)")
    ap.add_argument("--snps", type=int, default=None, help="override m per rank (testing only)")
    ap.add_argument("--overlap", type=int, default=1, help="1: pipeline block b's K2/K3 beside block b+1's K1")
    ap.add_argument("--fuse-k2", type=int, default=1, help="1: K2 fused into K1's epilogue for few traits (NEXT-2)")
    ap.add_argument("--kernel-steps", type=int, default=1, help="serial passes timed per kernel (roofline)")
    ap.add_argument("--no-chol-alt", dest="chol_alt", action="store_false",
                    help="skip the CLAK-Chol (Alg. 3) modes reported under `modes` for single-trait configs")
    ap.add_argument("--int8-slices", type=int, default=7, choices=(7, 8),
                    help="digits per fp64 value in the int8-sliced modes (8: <= 2^-57 representation error, 7: 2^-50)")
    ap.add_argument("--no-int8-alt", dest="int8_alt", action="store_false",
                    help="skip the int8-sliced mode measurement reported under `modes`")
    ap.add_argument("--no-lowrank-alt", dest="lowrank_alt", action="store_false",
                    help="skip the low-rank trait-weight modes (reading L1) reported under `modes` for t >= 16")
    ap.add_argument("--no-est-alt", dest="est_alt", action="store_false",
                    help="skip the variance-component estimation measurement reported under `modes.estimate`")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--check", type=int, default=2000, help="oracle spot-check pairs after timing (0 = off)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-traits", type=int, default=4)
    ap.add_argument("--cpu-snps", type=int, default=1024)
    ap.add_argument("--ref-snps", type=int, default=1024)
    args = ap.parse_args(argv)
    rank, world, _ = dist_env()
    if world != args.gpus and rank == 0:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    res = run_reference(args) if args.impl == "reference" else run_ours(args)
    if res is not None and rank == 0:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
