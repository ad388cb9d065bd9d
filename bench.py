#!/usr/bin/env python
"""Benchmark of the B200-native CLAK-Eig GLS-sequence hot path (BASELINE.json metric: GLS/s = SNP x trait pairs
per second, with the FP64 tensor-pipe fraction of peak).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

With --gpus N > 1 and no torchrun environment, bench.py re-launches itself through `torch.distributed.run` with N
ranks (one process per GPU, NCCL over NVLink) and fails loudly if fewer than N GPUs are visible; under torchrun it
checks that WORLD_SIZE == --gpus.  Never a silent 1-rank run labelled N.

A step = one pass of the whole hot path (Alg. 4 line 3 + lines 13-16: K1 rotation
GEMM, K2 weighted-reduction GEMM, K3 Schur solve) over every SNP of the rank's shard, for all t traits.
Setup (dsyevd, precompute, the one NCCL broadcast of the replicated state) is timed and reported separately.
Scaling: strong by default -- the config's m SNPs are split into N contiguous ranges, rank r
taking [r m / N, (r+1) m / N), so `value` = m t / (max over ranks of the step time).  `--scaling weak` (opt-in)
gives every rank its own m SNPs of an N m-SNP genome.

`value`: X_R already resident in HBM (uint8 dosages, exact), K1/K2 on the FP64 DMMA pipe (the north star's
         design), blocks pipelined over two streams; timed with CUDA events on the compute stream.
`e2e`:   the same through the public API from pinned HOST X_R (block staging on the copy stream inside the timed
         region) plus the device->host stream of every step's b, Var and status into pinned host memory.
`roofline`: the dominant kernel (K1, or K1 with K2 fused into its epilogue for few traits) from a serial pass of
         the same run (CUDA events around every launch; overlapped launches would share SMs).
`parity`: a stratified seeded subsample (reading A18, >= 10^4 pairs per rank, forced shard and block edges) is
         cut from EVERY rank's outputs of every mode, gathered on rank 0 and checked against the CPU oracle.
`modes`: the int8-sliced tcgen05 mode (NEXT-4), CLAK-Chol (t = 1, NEXT-1), estimation (NEXT-3) on the same inputs.
`--impl reference`: the CPU oracle (oracle/), as it stands, on a bounded sample of the same workload (rank 0).
"""
from __future__ import annotations

import argparse
import contextlib
import json
import os
import socket
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

# The paper's own CPU timings, quoted with their hardware (context, not the target).
PAPER_CONTEXT = {
    "hardware": "2x Intel Xeon X5675 (2 x 6 cores, 3.06 GHz, ~147 GFLOP/s fp64 peak), 96 GB RAM, MKL 10.3 + "
                "OpenMP, AIO double buffering (PAPER.md P:209-210)",
    "clak_eig_scenario_C": "n = 1 000, m = 1e6, 'thousands and more traits': 'from several months down to two "
                           "days'; 105x / 177x / 418x over GWFGLS / FaST-LMM / EMMAX (P:349-351) -- "
                           "5.8e3 GLS/s at t = 1e3 if two days (derived, BASELINE.md)",
    "transcriptome": "26 days on one node, 20 h on a 32-node cluster (P:288)",
    "clak_chol_single_trait": "n = 1 000, m = 1e7, t = 1: 2.5 min (P:343) = 6.7e4 GLS/s (derived); "
                              "n = 40 000: 35 h (P:343)",
}


# ------------------------------------------------------------------ host-side helpers (CPU-testable)
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def shard_range(m: int, rank: int, world: int, scaling: str = "strong"):
    """SNP columns of a rank.  strong: contiguous split of m; weak: [rank*m, (rank+1)*m) of an N*m genome."""
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


def parity_edges(m_rank: int, world: int, scaling: str, block: int):
    """SNPs every parity subsample must contain (reading A18): each shard's first and last SNP and the first and
    last SNP of the shard's blocks 0, 1 and final (short) block -- where block/shard arithmetic could go wrong."""
    forced = []
    for r in range(world):
        lo, hi = shard_range(m_rank, r, world, scaling)
        if hi <= lo:
            continue
        forced += [lo, hi - 1]
        last = (hi - lo - 1) // block * block
        for b0 in (0, block, last):
            for c in (lo + b0, lo + b0 + block - 1):
                if lo <= c < hi:
                    forced.append(c)
    return sorted(set(forced))


def parity_subsample(gcfg, m_rank: int, world: int, scaling: str, block: int, pairs_per_rank: int):
    """(snps, traits): the stratified seeded subsample of reading A18 over the whole (gathered) job, sized to
    >= pairs_per_rank pairs per rank, with parity_edges forced."""
    return datagen.subsample(gcfg, n_pairs=pairs_per_rank * world,
                             forced_snps=parity_edges(m_rank, world, scaling, block))


def local_pairs(snps, lo: int, hi: int):
    """Positions of the subsample SNPs that live in this rank's shard [lo, hi), as (global, local) int64 arrays."""
    sel = (snps >= lo) & (snps < hi)
    return snps[sel], snps[sel] - lo


def merge_gathered(parts, snps):
    """Rank 0: concatenate the ranks' (global_snps, {mode: (b, v, s)}) in SNP order and check the union covers the
    subsample exactly once.  Returns {mode: (b, v, s)} aligned with `snps`."""
    glob = np.concatenate([p["snps"] for p in parts]) if parts else np.zeros(0, np.int64)
    order = np.argsort(glob, kind="stable")
    if not np.array_equal(glob[order], snps):
        raise AssertionError("gathered parity subsample does not cover the subsample exactly once")
    modes = parts[0]["res"].keys()
    out = {}
    for mode in modes:
        cat = [np.concatenate([p["res"][mode][q] for p in parts])[order] for q in range(3)]
        out[mode] = tuple(cat)
    return out


def flops_per_block(n, p, t, cols):
    """Algorithmic flops: K1 2 n^2 k, K2 2 n k t (p+2); K3 ~ k t (p^2 + 4p + 8)."""
    return {"K1": 2.0 * n * n * cols, "K2": 2.0 * n * cols * t * (p + 2), "K3": cols * t * (p * p + 4 * p + 8.0)}


def k3_bytes(p, t, cols, full=False):
    """K3 algorithmic HBM bytes: reads 8 (p+2) per pair, writes 8+8+1 (SNP mode) or 16 (p+1)+1 (full)."""
    w = p + 1
    return cols * t * (8 * (p + 2) + (16 * w + 1 if full else 17))


def blocks_of(ncols: int, block: int):
    return [min(block, ncols - c) for c in range(0, ncols, block)]


def nvml_id(device) -> str:
    """The nvidia-smi / NVML identifier of a torch CUDA device: its UUID ("GPU-..."), because CUDA's device order
    (and CUDA_VISIBLE_DEVICES) need not match NVML's PCI order on a multi-GPU node; the CUDA ordinal as a fallback."""
    try:
        import torch
        u = str(torch.cuda.get_device_properties(device).uuid)
        if u:
            return u if u.startswith("GPU-") else "GPU-" + u
    except Exception:
        pass
    return str(device.index if hasattr(device, "index") else device)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms while the timed region runs, for one GPU or -- on rank 0
    of a multi-GPU run -- every rank's GPU in one query (`index`: an nvml_id or a list of them)."""
    FIELDS = "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap,uuid"

    def __init__(self, index):
        ids = [str(x) for x in index] if isinstance(index, (list, tuple)) else [str(index)]
        self.ids = list(dict.fromkeys(ids))  # ranks sharing a GPU (gloo test mode) query it once
        self.rows = []
        self._stop = threading.Event()
        self._th = None

    def _loop(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", ",".join(self.ids), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5).stdout
                for ln in out.strip().splitlines():
                    vals = [v.strip() for v in ln.split(",")]
                    if len(vals) >= 9:
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

    @staticmethod
    def _num(x):
        try:
            return float(x)
        except ValueError:
            return None

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

        def summ(rows):
            sm = [v for v in (self._num(r[0]) for r in rows) if v is not None]
            smax = [v for v in (self._num(r[1]) for r in rows) if v is not None]
            pw = [v for v in (self._num(r[2]) for r in rows) if v is not None]
            counts = {names[i]: sum(1 for r in rows if r[4 + i].lower().startswith("active")) for i in range(4)}
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                    "reasons": sorted(k for k, v in counts.items() if v),
                    "reason_samples": {k: v for k, v in counts.items() if v}, "samples": len(rows),
                    "power_w_max": max(pw) if pw else None}

        out = summ(self.rows)
        gpus = sorted({r[8] for r in self.rows})
        if len(gpus) > 1:  # multi-GPU: the slowest GPU's median and each GPU's own summary
            per = {g: summ([r for r in self.rows if r[8] == g]) for g in gpus}
            out["sm_mhz"] = min(v["sm_mhz"] for v in per.values() if v["sm_mhz"] is not None)
            out["per_gpu"] = per
        return out


class PcieSampler:
    """Device PCIe counters while the e2e region runs (NVML nvmlDeviceGetPcieThroughput: bytes over a 20 ms window,
    polled back to back in a thread): counter evidence for the block staging (H2D = RX, D2H = TX) beside the
    copy-event timing.  The mean over the windows estimates the average rate of the bursty copies."""

    def __init__(self, index):
        self.index = index  # nvml_id(): UUID or ordinal
        self.rx, self.tx = [], []
        self._stop = threading.Event()
        self._th = None
        self.err = None

    def _loop(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = (pynvml.nvmlDeviceGetHandleByUUID(self.index) if str(self.index).startswith("GPU-")
                 else pynvml.nvmlDeviceGetHandleByIndex(int(self.index)))
            self.link = {"gen": pynvml.nvmlDeviceGetCurrPcieLinkGeneration(h),
                         "width": pynvml.nvmlDeviceGetCurrPcieLinkWidth(h)}
            while not self._stop.is_set():
                self.rx.append(pynvml.nvmlDeviceGetPcieThroughput(h, pynvml.NVML_PCIE_UTIL_RX_BYTES))
                self.tx.append(pynvml.nvmlDeviceGetPcieThroughput(h, pynvml.NVML_PCIE_UTIL_TX_BYTES))
        except Exception as exc:  # no NVML: report why
            self.err = repr(exc)

    def __enter__(self):
        self.link = None
        self._th = threading.Thread(target=self._loop, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._th:
            self._th.join(timeout=10)

    def summary(self):
        if not self.rx:
            return {"samples": 0, "note": self.err or "no NVML samples"}
        kb = 1e3 / 1e9  # NVML reports KB/s
        return {"samples": len(self.rx), "link": self.link,
                "rx_h2d_gbs_mean": statistics.fmean(self.rx) * kb, "rx_h2d_gbs_max": max(self.rx) * kb,
                "tx_d2h_gbs_mean": statistics.fmean(self.tx) * kb, "tx_d2h_gbs_max": max(self.tx) * kb,
                "source": "NVML nvmlDeviceGetPcieThroughput (device PCIe counters, 20 ms windows back to back)"}


def fp64_peak():
    """FP64 DMMA peak, BUILDER-measured (MEASURED_PEAKS.json, driver-written, has no FP64 entry):
    tools/fp64_peak.cu, back-to-back mma.sync.m8n8k4.f64 on all SMs (profiles/fp64_peak_r01.json).  It agrees with
    148 SM x 128 flop/clk x 1.965 GHz = 37.2 TF."""
    with open(os.path.join(ROOT, "profiles", "fp64_peak_r01.json")) as f:
        d = json.load(f)
    return float(d["dmma_tflops"]), ("builder-measured, not driver-written: tools/fp64_peak.cu DMMA.8x8x4 "
                                     "microbenchmark (profiles/fp64_peak_r01.json); theoretical 148 x 128 flop/clk "
                                     "x 1.965 GHz = 37.2 TF")


def i8_peak():
    """kind::i8 tcgen05 peak, builder-measured (tools/umma_i8_peak.cu, operands resident in shared memory,
    profiles/umma_i8_peak_r01.log): the best case of the MMA shapes the int8 kernel issues."""
    best = 0.0
    with open(os.path.join(ROOT, "profiles", "umma_i8_peak_r01.log")) as f:
        for ln in f:
            ln = ln.strip()
            if ln.startswith("{"):
                best = max(best, float(json.loads(ln)["tops"]))
    return best, ("builder-measured: tools/umma_i8_peak.cu tcgen05.mma kind::i8 M128 with smem-resident operands "
                  "(profiles/umma_i8_peak_r01.log, best case); MEASURED_PEAKS.json has no int8 entry")


def ncu_traffic(n, block, fused, int8):
    """DRAM bytes per launch of the dominant kernel from an ncu --set full capture of the SAME shape
    (profiles/k1_traffic.json entries keyed by n, block_cols, fused, int8), else None."""
    path = os.path.join(ROOT, "profiles", "k1_traffic.json")
    if not os.path.exists(path):
        return None, None
    with open(path) as f:
        d = json.load(f)
    for e in d.get("entries", []):
        if (e["n"], e["block_cols"], bool(e["fused"]), int(e["int8"])) == (n, block, bool(fused), int(int8)):
            return e["bytes_per_launch"], e["source"]
    return None, None


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


# ------------------------------------------------------------------ oracle (cpu_baseline / --impl reference)
def all_host_cores():
    """The oracle runs on all of the host's cores: torch.distributed.run sets OMP_NUM_THREADS=1 in every rank, which
    would otherwise leave rank 0's LAPACK (parity check, cpu_baseline, the reference arm) on one thread."""
    import threadpoolctl
    return threadpoolctl.threadpool_limits(limits=host_cores())


def _blas_threads():
    import threadpoolctl
    info = threadpoolctl.threadpool_info()
    return max([i.get("num_threads", 1) for i in info] or [1])


def oracle_sample(cfg, ds, traits, snps):
    """Time the CPU oracle, as it stands (trait-cached: Alg. 1 lines 1-2 once per trait), on (snps x traits) of the
    config.  Returns (pairs, seconds, threads)."""
    import scipy.linalg  # noqa: F401  (loads the LAPACK the oracle uses)

    import oracle
    G = datagen.xr_columns(cfg, snps)
    t0 = time.perf_counter()
    oracle.gls_sequence(ds.Phi, ds.XL, G, ds.Y, ds.h2, ds.s2, traits=traits)
    dt = time.perf_counter() - t0
    return len(snps) * len(traits), dt, _blas_threads()


def oracle_literal_sample(cfg, ds, pairs, budget_s):
    """Time the oracle's LITERAL mode -- Alg. 1 per (i, j) with M_j assembled and Cholesky-factored for every pair,
    Table 1's 'Naive' O(m t n^3) row -- on seeded pairs until `budget_s` seconds have elapsed.
    Returns (pairs_done, seconds, threads)."""
    import oracle
    G = datagen.xr_columns(cfg, [i for i, _ in pairs])
    t0 = time.perf_counter()
    done = 0
    for c, (_, j) in enumerate(pairs):
        oracle.gls_single(ds.Phi, np.column_stack([ds.XL, G[:, c]]), ds.Y[:, j], ds.s2[j], ds.h2[j])
        done += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    return done, time.perf_counter() - t0, _blas_threads()


def cpu_baseline(cfg, ds, args):
    rng = np.random.default_rng(cfg.seed)
    traits = np.sort(rng.choice(cfg.t, size=min(cfg.t, args.cpu_traits), replace=False))
    snps = np.sort(rng.choice(cfg.m, size=min(cfg.m, args.cpu_snps), replace=False))
    pairs, sec, thr = oracle_sample(cfg, ds, traits, snps)
    lit_pairs = [(int(rng.integers(cfg.m)), int(rng.integers(cfg.t))) for _ in range(64)]
    lp, ls, lthr = oracle_literal_sample(cfg, ds, lit_pairs, args.cpu_literal_s)
    return {"value": pairs / sec, "unit": UNIT, "cores": thr, "kind": "oracle",
            "sample": f"{pairs} pairs of {cfg.name} ({len(traits)} traits x {len(snps)} SNPs), trait-cached "
                      f"Alg. 1 (M_j factored once per trait), fp64 numpy/LAPACK, {sec:.1f} s",
            "cpu_model": cpu_model(), "host_cores": host_cores(),
            "projected_full_config_s": cfg.m * cfg.t / (pairs / sec),
            "literal": {"value": lp / ls, "unit": UNIT, "cores": lthr, "pairs": lp, "seconds": ls,
                        "what": "Alg. 1 per (i, j), M_j re-assembled and re-factored per pair (Table 1 'Naive', "
                                "P:193)", "projected_full_config_s": cfg.m * cfg.t / (lp / ls)},
            "paper_context": PAPER_CONTEXT}


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


def _nccl_lines(rank):
    """This rank's NCCL INIT log lines (communicator size, topology) written to NCCL_DEBUG_FILE."""
    path = os.environ.get("GWAS_NCCL_LOG")
    if not path or not os.path.exists(path):
        return []
    with open(path, errors="replace") as f:
        lines = [ln.rstrip() for ln in f if ("nRanks" in ln or "Init COMPLETE" in ln or "NVLS" in ln)]
    for ln in lines:
        print(f"[rank {rank}] {ln}", file=sys.stderr, flush=True)
    return lines[:8]


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    # GWAS_BENCH_BACKEND=gloo (testing only): exercise the multi-rank path (broadcast + attach, max over ranks) with
    # all ranks on the visible GPU(s); NCCL needs one GPU per rank.  Numbers from such a run are not bench values.
    backend = os.environ.get("GWAS_BENCH_BACKEND", "nccl")
    if backend == "nccl" and world > 1 and torch.cuda.device_count() < world:
        raise SystemExit(f"bench.py: {world} NCCL ranks need {world} GPUs, {torch.cuda.device_count()} visible")
    local = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            # NCCL prints its communicator lines (nRanks, NVLS) to a per-rank file; they go to stderr and the JSON
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            if "NCCL_DEBUG_FILE" not in os.environ:
                os.environ["NCCL_DEBUG_FILE"] = f"/tmp/gwas_bench_nccl.r{rank}.{os.getpid()}.log"
                os.environ["GWAS_NCCL_LOG"] = os.environ["NCCL_DEBUG_FILE"]
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    import paper_1207_2169_b200 as gw

    cfg = datagen.CONFIGS[args.config]
    m_rank = cfg.m if args.snps is None else args.snps
    lo, hi = shard_range(m_rank, rank, world, args.scaling)
    m_total = m_rank * world if args.scaling == "weak" else m_rank
    gcfg = datagen.Config(cfg.index, cfg.n, cfg.p, m_total, cfg.t, cfg.S, cfg.h2_range, cfg.s2_range)
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

    def make_engine(i8, overlap, algorithm="eig", block=args.block):
        """Rank 0 sets up (eig + precompute), the state is replicated by ONE broadcast, other ranks attach."""
        eng = gw.Gwas(n, p, t, device=local, block_cols=block, timing=True, int8_slices=i8, overlap=overlap,
                      algorithm=algorithm, fuse_k2=bool(args.fuse_k2))
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
            info["ms_broadcast"] = max_over_ranks(e0.elapsed_time(e1), world, dev)
            info["broadcast_bytes"] = eng.state_bytes
            info["broadcast_gbs"] = eng.state_bytes / (info["ms_broadcast"] / 1e3) / 1e9
            if rank != 0:
                eng.attach()
        # a second, serial context on the same state (gwas_attach) times the kernels one by one
        ser = gw.Gwas(n, p, t, device=local, block_cols=block, timing=True, int8_slices=i8, overlap=False,
                      algorithm=algorithm, fuse_k2=bool(args.fuse_k2))
        ser.state.copy_(eng.state)
        ser.attach()
        info.update(eng.run_info())
        return eng, ser, info

    xr_dev = xr_host.to(dev)
    peak, peak_src = fp64_peak()
    nccl = _nccl_lines(rank) if world > 1 else []

    # ---------------- parity subsample: every rank cuts its own SNPs out of every mode's outputs
    local_res = {}
    sub = None
    glob_snps = loc_snps = None

    def cut(name, out):
        if sub is None:
            return
        b, v, s = out
        if b.is_cuda:
            torch.cuda.synchronize(dev)
            li = torch.from_numpy(loc_snps).to(dev)
            ti = torch.from_numpy(sub[1]).to(dev)
            local_res[name] = tuple(x.index_select(0, li).index_select(1, ti).cpu().numpy() for x in (b, v, s))
        else:
            torch.cuda.synchronize(dev)
            local_res[name] = tuple(x.numpy()[np.ix_(loc_snps, sub[1])].copy() for x in (b, v, s))

    # ================= headline mode: FP64 DMMA (the north star's K1/K2) =================
    eng, ser, setup = make_engine(0, bool(args.overlap))
    block = setup["block_cols"]
    fused = setup["fused_k2"]
    if args.check:
        sub = parity_subsample(gcfg, m_rank, world, args.scaling, block, args.check)
        glob_snps, loc_snps = local_pairs(sub[0], lo, hi)
    out = eng.alloc_outputs(ncols)
    stream = eng.compute_stream
    for _ in range(args.warmup):
        eng.run(xr_dev, out=out)
    if world > 1:  # rank 0 samples every rank's GPU in one nvidia-smi query (one sampler per node, not per rank)
        ids = [None] * world
        dist.all_gather_object(ids, nvml_id(dev))
    else:
        ids = [nvml_id(dev)]
    with (ClockSampler(ids) if rank == 0 else contextlib.nullcontext()) as clk:
        ms = _timed_steps(eng, xr_dev, out, args.steps, stream, barrier)
    ms_max = max_over_ranks(ms, world, dev)
    pairs_total = float(m_total) * t
    value = pairs_total * args.steps / (ms_max / 1e3)
    cut("fp64", out)
    blocks = blocks_of(ncols, block)
    fl = [flops_per_block(n, p, t, c) for c in blocks]
    k1_flops = sum(f["K1"] for f in fl)
    k2_flops = sum(f["K2"] for f in fl)
    kt = _kernel_pass(ser, xr_dev, out, args.kernel_steps, barrier)
    k1_ms, k2_ms, k3_ms = (kt[k]["ms"] / args.kernel_steps for k in ("K1", "K2", "K3"))
    k1_launches = max(1, kt["K1"]["launches"] // args.kernel_steps)
    serial_ms = k1_ms + k2_ms + k3_ms
    k3_gbs = sum(k3_bytes(p, t, c) for c in blocks) / (k3_ms / 1e3) / 1e9
    if fused:
        # K2 is contracted in K1's epilogue (NEXT-2): one fused stage; the K2 timer covers only the fixed-order
        # reduction of the per-tile partials (fused_k2_reduce)
        dom_flops, dom_name = k1_flops + k2_flops, "K1 with K2 fused in its epilogue (FP64 DMMA + epilogue DFMA)"
        stages = {"K1K2_fused_tflops": (k1_flops + k2_flops) / (k1_ms / 1e3) / 1e12,
                  "K1K2_fused_frac_of_peak": (k1_flops + k2_flops) / (k1_ms / 1e3) / 1e12 / peak,
                  "K2_reduce_ms_per_step": k2_ms,
                  "K1K2_incl_reduce_tflops": (k1_flops + k2_flops) / ((k1_ms + k2_ms) / 1e3) / 1e12,
                  "K3_hbm_gbs": k3_gbs,
                  "share_of_serial_step": {"K1+K2 fused": k1_ms / serial_ms, "K2 reduce": k2_ms / serial_ms,
                                           "K3": k3_ms / serial_ms}}
    else:
        dom_flops, dom_name = k1_flops, "K1 rotation GEMM (FP64 DMMA)"
        k1_tf = k1_flops / (k1_ms / 1e3) / 1e12
        k2_tf = k2_flops / (k2_ms / 1e3) / 1e12
        gemm_tf = (k1_flops + k2_flops) / ((k1_ms + k2_ms) / 1e3) / 1e12
        stages = {"K1_tflops": k1_tf, "K1_frac_of_peak": k1_tf / peak, "K2_tflops": k2_tf,
                  "K2_frac_of_peak": k2_tf / peak, "K1K2_tflops": gemm_tf, "K1K2_frac_of_peak": gemm_tf / peak,
                  "K3_hbm_gbs": k3_gbs,
                  "share_of_serial_step": {"K1": k1_ms / serial_ms, "K2": k2_ms / serial_ms, "K3": k3_ms / serial_ms}}
    dom_tf = dom_flops / (k1_ms / 1e3) / 1e12
    traffic, traffic_src = ncu_traffic(n, block, fused, 0)
    step_tf = (k1_flops + k2_flops) * args.steps / (ms / 1e3) / 1e12

    # e2e through the public API: pinned host X_R in, pinned host (b, var, status) out -- the library stages
    # blocks H2D and streams each block's results D2H while later blocks compute
    b_h, v_h, s_h = eng.alloc_outputs(ncols, host=True)
    e2e_steps = max(1, args.e2e_steps)
    eng.run(xr_host, out=(b_h, v_h, s_h))
    barrier()
    eng.kernel_times(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with (PcieSampler(nvml_id(dev)) if rank == 0 else contextlib.nullcontext()) as pcie:
        e0.record(stream)
        for _ in range(e2e_steps):
            eng.run(xr_host, out=(b_h, v_h, s_h))
        e1.record(stream)
        barrier()
    ms_e2e_rank = e0.elapsed_time(e1)
    ms_e2e = max_over_ranks(ms_e2e_rank, world, dev)
    e2e_value = pairs_total * e2e_steps / (ms_e2e / 1e3)
    h2d = ((ncols - 1) * ld + n) if ncols else 0  # uint8 dosages copied per step (this rank)
    kt_e2e = eng.kernel_times(reset=True)  # H2D: CUDA events around every staging copy (copy stream)
    staging_gbs = h2d * e2e_steps / (kt_e2e["H2D"]["ms"] / 1e3) / 1e9 if kt_e2e["H2D"]["ms"] > 0 else None
    d2h = b_h.numel() * 8 + v_h.numel() * 8 + s_h.numel()
    cut("e2e_host", (b_h, v_h, s_h))
    eng.close()
    ser.close()
    del eng, ser, b_h, v_h, s_h

    # ================= int8-sliced mode, same inputs =================
    modes = {}
    if args.int8_alt:
        S = args.int8_slices
        eng8, ser8, setup8 = make_engine(S, True, block=8192)
        for _ in range(args.warmup):
            eng8.run(xr_dev, out=out)
        ms8 = max_over_ranks(_timed_steps(eng8, xr_dev, out, args.steps, eng8.compute_stream, barrier), world, dev)
        cut("int8_sliced", out)
        blocks8 = blocks_of(ncols, setup8["block_cols"])
        kt8 = _kernel_pass(ser8, xr_dev, out, args.kernel_steps, barrier)
        i1_ms, i2_ms, i3_ms = (kt8[k]["ms"] / args.kernel_steps for k in ("K1", "K2", "K3"))
        na_pad = (n + 63) // 64 * 64
        nlin_pad = (t * (p + 1) + 63) // 64 * 64
        i8_ops = sum(2.0 * c * (na_pad + nlin_pad) * S * n for c in blocks8)   # int8 MACs x 2 actually issued
        ipk, ipk_src = i8_peak()
        k2b_flops = sum(2.0 * n * c * t for c in blocks8)
        modes["int8_sliced"] = {
            "value": pairs_total * args.steps / (ms8 / 1e3), "unit": UNIT, "ms_per_step": ms8 / args.steps,
            "int8_slices": S, "representation_error": f"<= 2^-{7 * S + 1} of each digitised column's largest entry",
            "roofline": {"bound": "tensor", "kernel": f"K1i+K2a int8-sliced tcgen05 ({S} digits, TMEM int32)",
                         "achieved": i8_ops / (i1_ms / 1e3) / 1e12, "peak": ipk, "unit": "TOPS",
                         "frac": i8_ops / (i1_ms / 1e3) / 1e12 / ipk, "peak_source": ipk_src,
                         "fp64_equiv_tflops": (k1_flops + sum(2.0 * n * c * t * (p + 1) for c in blocks8))
                                              / (i1_ms / 1e3) / 1e12},
            "k2b_dmma_tflops": k2b_flops / (i2_ms / 1e3) / 1e12,
            "k2b_frac_of_fp64_peak": k2b_flops / (i2_ms / 1e3) / 1e12 / peak,
            "share_of_serial_step": {k: v / (i1_ms + i2_ms + i3_ms) for k, v in
                                     (("K1i+K2a", i1_ms), ("K2b", i2_ms), ("K3", i3_ms))},
            "setup": setup8}
        eng8.close()
        ser8.close()

    # ================= fp64 X_R staged from pinned host (the PCIe roofline; SURVEY §8(d) staging check) ==========
    # uint8 dosages are the default (1 byte per entry); with fp64 dosages (8 bytes) the small-n configs become
    # staging-bound: n = 1e3, t = 1 needs 8 KB per SNP over PCIe against 2n^2 = 2e6 flop of K1.  Only where the fp64
    # shard fits a modest pinned buffer (<= 8 GB).
    if args.f64_alt and ncols * ld * 8 <= 8e9:
        x64_h = torch.empty((ncols, ld), dtype=torch.float64, pin_memory=True)
        x64_h.copy_(xr_host)
        # the PCIe yardstick: plain pinned -> HBM copies of the same bytes in the same 8192-SNP pieces, back to back
        # on one stream (no compute), best of two passes
        probe = torch.empty((min(ncols, 8192), ld), dtype=torch.float64, device=dev)
        pcie_gbs = 0.0
        for _ in range(2):
            ep0, ep1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(dev)
            ep0.record()
            for c0 in range(0, ncols, 8192):
                c1 = min(ncols, c0 + 8192)
                probe[: c1 - c0].copy_(x64_h[c0:c1], non_blocking=True)
            ep1.record()
            torch.cuda.synchronize(dev)
            pcie_gbs = max(pcie_gbs, ncols * ld * 8 / (ep0.elapsed_time(ep1) / 1e3) / 1e9)
        del probe
        eng64 = gw.Gwas(n, p, t, device=local, block_cols=args.block, timing=True, overlap=True, xr_dtype="f64",
                        fuse_k2=bool(args.fuse_k2))
        if rank == 0:
            eng64.setup(ds.Phi, ds.XL, ds.Y, ds.h2, ds.s2)
        if world > 1:
            barrier()
            replicate_state(eng64.state, world)
            barrier()
            if rank != 0:
                eng64.attach()
        for _ in range(args.warmup):
            eng64.run(x64_h, out=out)
        eng64.kernel_times(reset=True)
        ms64 = max_over_ranks(_timed_steps(eng64, x64_h, out, args.steps, eng64.compute_stream, barrier), world, dev)
        kt64 = eng64.kernel_times(reset=True)
        cut("fp64_staged", out)
        h2d64 = ncols * ld * 8
        modes["fp64_staged"] = {
            "value": pairs_total * args.steps / (ms64 / 1e3), "unit": UNIT, "ms_per_step": ms64 / args.steps,
            "what": "X_R as fp64 dosages in pinned host memory, staged block by block on the copy stream (device "
                    "outputs), K1/K2 on FP64 DMMA",
            "roofline": {"bound": "pcie" if h2d64 / (ms64 / args.steps / 1e3) / 1e9 >= 0.8 * pcie_gbs
                         else "compute (staging hidden behind K1/K2)",
                         "achieved": h2d64 * world / (ms64 / args.steps / 1e3) / 1e9,
                         "peak": pcie_gbs, "unit": "GB/s",
                         "frac": h2d64 / (ms64 / args.steps / 1e3) / 1e9 / pcie_gbs,
                         "peak_source": "measured in this run: plain pinned-host -> HBM copies of the same bytes "
                                        "in 8192-SNP pieces, back to back, no compute"},
            "staging_h2d_gbs_events": h2d64 * args.steps / (kt64["H2D"]["ms"] / 1e3) / 1e9
            if kt64["H2D"]["ms"] > 0 else None,
            "h2d_bytes_per_step": h2d64 * world}
        eng64.close()
        del x64_h

    # ================= CLAK-Chol single-trait path (Alg. 3, NEXT-1), t == 1 only =================
    if t == 1 and args.chol_alt:
        for i8 in (0, args.int8_slices):
            engc, serc, setupc = make_engine(i8, True, "chol", block=args.block if i8 == 0 else 8192)
            for _ in range(args.warmup):
                engc.run(xr_dev, out=out)
            msc = max_over_ranks(_timed_steps(engc, xr_dev, out, args.steps, engc.compute_stream, barrier), world,
                                 dev)
            name = "chol_int8_sliced" if i8 else "chol_fp64"
            cut(name, out)
            ktc = _kernel_pass(serc, xr_dev, out, args.kernel_steps, barrier)
            c1_ms = ktc["K1"]["ms"] / args.kernel_steps
            tri_flops = sum(1.0 * n * n * c for c in blocks_of(ncols, setupc["block_cols"]))   # L^-1 X_R: n^2 k
            entry = {"value": pairs_total * args.steps / (msc / 1e3), "unit": UNIT, "ms_per_step": msc / args.steps,
                     "K1_ms_per_step": c1_ms, "setup": setupc,
                     "K1_tflops_algorithmic": tri_flops / (c1_ms / 1e3) / 1e12}
            if i8 == 0:
                entry["K1_frac_of_fp64_peak"] = entry["K1_tflops_algorithmic"] / peak
            modes[name] = entry
            engc.close()
            serc.close()

    # ================= low-rank trait weights (reading L1, outside §8): opt-in only =================
    if t >= 16 and args.lowrank_alt:
        for i8 in (0, args.int8_slices):
            engl = gw.Gwas(n, p, t, device=local, block_cols=8192, timing=True, int8_slices=i8, overlap=True,
                           trait_rank=-1)
            if rank == 0:
                engl.setup(ds.Phi, ds.XL, ds.Y, ds.h2, ds.s2)
            if world > 1:
                barrier()
                replicate_state(engl.state, world)
                barrier()
                if rank != 0:
                    engl.attach()
            for _ in range(args.warmup):
                engl.run(xr_dev, out=out)
            msl = max_over_ranks(_timed_steps(engl, xr_dev, out, args.steps, engl.compute_stream, barrier), world,
                                 dev)
            name = "lowrank_int8_sliced" if i8 else "lowrank_fp64"
            cut(name, out)
            modes[name] = {"value": pairs_total * args.steps / (msl / 1e3), "unit": UNIT,
                           "ms_per_step": msl / args.steps, "note": "reading L1: an approximation outside SURVEY §8"}
            engl.close()

    # ================= variance-component estimation (the paper's first step, NEXT-3) =================
    if args.est_alt and rank == 0:
        modes["estimate"] = bench_estimate(gw, cfg, ds, local, args)

    # ---------------- parity: gather every rank's subsample cut, check on rank 0 (outside timed regions)
    parity = None
    rank_info = {"rank": rank, "gpu": torch.cuda.get_device_name(dev),
                 "gpu_uuid": str(getattr(torch.cuda.get_device_properties(dev), "uuid", "")),
                 "shard": [lo, hi], "ms_per_step": ms / args.steps, "e2e_ms_per_step": ms_e2e_rank / e2e_steps,
                 "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "nccl_init": nccl}
    payload = {"snps": glob_snps if glob_snps is not None else np.zeros(0, np.int64), "res": local_res,
               "info": rank_info}
    if world > 1:
        parts = [None] * world
        dist.all_gather_object(parts, payload)
    else:
        parts = [payload]
    if args.check and rank == 0:
        with all_host_cores():
            parity = check_parity(gcfg, ds, sub, parts)
        for name, pr in list(parity["modes"].items()):
            if name in modes:
                modes[name]["parity"] = pr

    res = None
    if rank == 0:
        clocks = clk.summary()
        res = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic (datagen, seeded)",
            "config": {"workload": f"{cfg.name}: n={n}, p={p}, m={m_total}, t={t}, k={block}, "
                                   f"X_R uint8 dosages resident in HBM, K1/K2 FP64 DMMA",
                       "n": n, "p": p, "m": m_total, "t": t, "block_cols": block,
                       "block_cols_note": "auto (gwas_options.block_cols = 0): the k whose K1/K2 tile grids "
                                          "quantise best into whole waves" if args.block == 0 else "fixed",
                       "pairs_per_step": pairs_total, "parallelism": f"snp-shard x{world}",
                       "scaling": args.scaling, "shards": [p_["info"]["shard"] for p_ in parts],
                       "overlap": bool(args.overlap), "fused_k2": fused,
                       "l2": "inputs larger than L2 (Z 0.8 GB, X_R 10 GB at C4); no flush"},
            "roofline": {"bound": "tensor", "kernel": dom_name, "achieved": dom_tf,
                         "peak": peak, "unit": "TFLOP/s", "frac": dom_tf / peak, "traffic": traffic,
                         "traffic_source": traffic_src or "no ncu capture of this shape in profiles/k1_traffic.json",
                         "algorithmic_flops_per_launch": dom_flops / k1_launches,
                         "avg_launch_ms": k1_ms / k1_launches, "launches_per_step": k1_launches,
                         "timing": "CUDA events around every launch on the compute stream, serial pass of the "
                                   "same run (rank 0)",
                         "peak_source": peak_src},
            "gemm_stages": stages,
            "step_gemm_tflops": step_tf, "step_gemm_frac_of_peak": step_tf / peak,
            "e2e": {"value": e2e_value, "unit": UNIT,
                    "h2d_bytes_per_step": sum(p_["info"]["h2d_bytes_per_step"] for p_ in parts),
                    "d2h_bytes_per_step": sum(p_["info"]["d2h_bytes_per_step"] for p_ in parts), "steps": e2e_steps, "ms_per_step": ms_e2e / e2e_steps,
                    "staging_h2d_gbs": staging_gbs,
                    "pcie_counters": pcie.summary(),
                    "avg_h2d_gbs": h2d / (ms_e2e_rank / e2e_steps / 1e3) / 1e9,
                    "avg_d2h_gbs": d2h / (ms_e2e_rank / e2e_steps / 1e3) / 1e9,
                    "staging_note": "pinned host -> HBM block copies on the copy stream (PCIe), timed by CUDA events "
                                    "around each copy while compute runs (rank 0)"},
            "gpu_launches": 3 * len(blocks) * args.steps,
            "setup": {**setup, "datagen_s": t_gen},
            "ranks": [p_["info"] for p_ in parts],
            "clocks": clocks,
        }
        if modes:
            res["modes"] = modes
        if parity is not None:
            res["parity"] = {k: v for k, v in parity.items() if k != "modes"}
        if not args.no_cpu_baseline:
            with all_host_cores():
                res["cpu_baseline"] = cpu_baseline(cfg, ds, args)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return res


def check_parity(gcfg, ds, sub, parts):
    """Rank 0: the oracle on the gathered subsample; every mode's outputs from every rank against it."""
    import oracle
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from gpu_helpers import TOL_B, TOL_VAR, compare
    snps, traits = sub
    merged = merge_gathered(parts, snps)
    G = datagen.xr_columns(gcfg, snps)
    t0 = time.perf_counter()
    ref = oracle.gls_sequence(ds.Phi, ds.XL, G, ds.Y, ds.h2, ds.s2, traits=traits)
    t_oracle = time.perf_counter() - t0
    out = {"modes": {}}
    for name, (b, v, s) in merged.items():
        eb, ev = compare(b, v, s, ref)
        per_rank = []
        for p_ in parts:
            sel = np.isin(snps, p_["snps"])
            if sel.any():
                rb = {"b": ref["b"][sel], "Var": ref["Var"][sel], "status": ref["status"][sel]}
                e1, e2 = compare(b[sel], v[sel], s[sel], rb)
                per_rank.append({"rank": p_["info"]["rank"], "pairs": int(sel.sum() * traits.size),
                                 "max_db_over_se": e1, "max_var_rel": e2})
        out["modes"][name] = {"pairs": int(snps.size * traits.size), "max_db_over_se": eb, "max_var_rel": ev,
                              "tol": TOL_B, "pass": bool(eb <= TOL_B and ev <= TOL_VAR), "per_rank": per_rank}
    head = out["modes"]["fp64"]
    out.update({"pairs": head["pairs"], "snps": int(snps.size), "traits": int(traits.size),
                "max_db_over_se": head["max_db_over_se"], "max_var_rel": head["max_var_rel"], "tol": TOL_B,
                "pass": all(m["pass"] for m in out["modes"].values()),
                "per_rank": head["per_rank"], "e2e_host": out["modes"]["e2e_host"],
                "oracle_s": t_oracle, "what": "reading A18 stratified subsample, shard / block edges forced, "
                                             "cut from every rank's outputs and gathered on rank 0"})
    return out


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
        eng = gw.Gwas(cfg.n, cfg.p, cfg.t, device=local, block_cols=8192)
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
        with all_host_cores():
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
                             "sample": f"per step 1 trait x {args.ref_snps} SNPs of {cfg.name}, trait-cached Alg. 1; "
                                       f"{host_cores()} host cores ({cpu_model()})"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


# ------------------------------------------------------------------ launcher
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def self_launch(args, argv):
    """--gpus N > 1 without a torchrun environment: re-run this script under torch.distributed.run with N ranks on
    this node (127.0.0.1 rendezvous).  Fails loudly when N NCCL ranks cannot each get a GPU."""
    backend = os.environ.get("GWAS_BENCH_BACKEND", "nccl")
    if args.impl == "ours" and backend == "nccl":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs (one NCCL rank per GPU); {have} visible",
                  file=sys.stderr, flush=True)
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *argv]
    print("bench.py: launching " + " ".join(cmd[1:]), file=sys.stderr, flush=True)
    return subprocess.call(cmd, env=dict(os.environ))


def build_parser():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4, help="BASELINE.json config index (default 4)")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="strong (default): split the config's m SNPs over the ranks; weak: m SNPs per rank")
    ap.add_argument("--block", type=int, default=0,
                    help="SNP columns per streamed block k (0 = auto: whole-wave quantisation of K1/K2)")
    ap.add_argument("--snps", type=int, default=None, help="override m (testing only)")
    ap.add_argument("--overlap", type=int, default=1, help="1: pipeline block b's K2/K3 beside block b+1's K1")
    ap.add_argument("--fuse-k2", type=int, default=1, help="1: K2 fused into K1's epilogue for few traits (NEXT-2)")
    ap.add_argument("--kernel-steps", type=int, default=1, help="serial passes timed per kernel (roofline)")
    ap.add_argument("--no-chol-alt", dest="chol_alt", action="store_false",
                    help="skip the CLAK-Chol (Alg. 3) modes reported under `modes` for single-trait configs")
    ap.add_argument("--int8-slices", type=int, default=7, choices=(7, 8),
                    help="digits per fp64 value in the int8-sliced modes (8: <= 2^-57 representation error, 7: 2^-50)")
    ap.add_argument("--no-int8-alt", dest="int8_alt", action="store_false",
                    help="skip the int8-sliced mode measurement reported under `modes`")
    ap.add_argument("--lowrank-alt", dest="lowrank_alt", action="store_true",
                    help="also time the low-rank trait-weight modes (reading L1, outside SURVEY §8) for t >= 16")
    ap.add_argument("--no-f64-alt", dest="f64_alt", action="store_false",
                    help="skip the fp64-dosage staged run (`modes.fp64_staged`, PCIe roofline; shards <= 8 GB in fp64)")
    ap.add_argument("--no-est-alt", dest="est_alt", action="store_false",
                    help="skip the variance-component estimation measurement reported under `modes.estimate`")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--check", type=int, default=10_000,
                    help="oracle parity pairs per rank, cut from every mode's outputs after timing (0 = off)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-traits", type=int, default=4)
    ap.add_argument("--cpu-snps", type=int, default=1024)
    ap.add_argument("--cpu-literal-s", type=float, default=5.0, help="seconds of the oracle's literal per-pair mode")
    ap.add_argument("--ref-snps", type=int, default=1024)
    return ap


def main(argv=None):
    argv = sys.argv[1:] if argv is None else list(argv)
    args = build_parser().parse_args(argv)
    rank, world, _ = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(self_launch(args, argv))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: refusing to report a mislabelled run",
              file=sys.stderr, flush=True)
        sys.exit(2)
    res = run_reference(args) if args.impl == "reference" else run_ours(args)
    if res is not None and rank == 0:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
