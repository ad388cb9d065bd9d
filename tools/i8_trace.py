"""Summarise GWAS_I8_TRACE phase stamps of the int8 kernel (debug).  Usage: python tools/i8_trace.py trace.bin
Slots per CTA (16): 0 entry, 1 after TMEM alloc + barrier init, 2 first stage landed (MMA thread), 3 last commit
issued, 4 epilogue sees accumulators, 5 epilogue done, 6 before dealloc, 7 smid, 8 clock64 cycles the MMA thread
waited on full barriers (after the first stage), 9 cycles the producer waited on empty barriers, 10 k-stages.
Persistent 2-SM kernel: slots 2 / 3 bracket ALL of a CTA's tiles and slot 10 counts all its k-stages, so "mainloop
per k-stage" is the CTA's average stage time with the epilogues included; slot 4 is the last tile's drain start."""
import sys
import numpy as np
a = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 4096, 16)
for li, L in enumerate(a):
    v = L[L[:, 0] > 0].astype(np.int64)
    if not len(v):
        continue
    t0 = v[:, 0].min()
    def d(i, j):
        ok = (v[:, i] > 0) & (v[:, j] > 0)  # 2-SM kernel: only the pair's leader stamps the MMA phases
        return np.median(v[ok, j] - v[ok, i]) / 1e3 if ok.any() else float("nan")
    print(f"launch {li}: {len(v)} CTAs, span {(v[:, 6].max() - t0) / 1e3:.1f} us; median us: setup {d(0, 1):.2f} "
          f"first-data {d(1, 2):.2f} mainloop {d(2, 3):.2f} commit->epi {d(3, 4):.2f} epilogue {d(4, 5):.2f} "
          f"tail {d(5, 6):.2f} total {d(0, 6):.2f}")
    mma = v[v[:, 10] > 0]
    if len(mma):
        ml = (mma[:, 3] - mma[:, 2]) * 1.965e3 / 1e3  # ns -> cycles at 1965 MHz
        print(f"   per k-stage (median): mainloop {np.median(ml / mma[:, 10]):.0f} cyc, MMA thread waiting on full "
              f"{np.median(mma[:, 8] / mma[:, 10]):.0f} cyc, producer waiting on empty {np.median(v[:, 9] / np.maximum(v[:, 10], 1)):.0f} cyc")
    gaps = []
    for sm in np.unique(v[:, 7]):
        w = v[v[:, 7] == sm]
        w = w[np.argsort(w[:, 0])]
        gaps += list((w[1:, 0] - w[:-1, 6]) / 1e3)
    if gaps:
        print(f"   launch gap between CTAs on one SM: median {np.median(gaps):.2f} us, p90 {np.percentile(gaps, 90):.2f}")
