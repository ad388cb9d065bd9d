"""Shared helpers for the -m gpu parity tests (GPU path through the C-ABI vs the CPU oracle)."""
import numpy as np

TOL_B = 1e-8     # max |b_gpu - b_ref| / SE_ref   (BASELINE.json north_star)
TOL_VAR = 1e-8   # max |Var_gpu - Var_ref| / Var_ref


def compare(b, v, st, ref, full=False):
    """b, v, st: GPU results for the pairs of `ref` (numpy, [i][j] or [i][j][e]).  Returns (err_b, err_var)
    and asserts statuses match exactly."""
    rst = ref["status"]
    assert st.shape == rst.shape
    mism = np.argwhere(st != rst)
    assert mism.size == 0, f"status mismatch at {mism[:5].tolist()} gpu={st[tuple(mism[0])]} ref={rst[tuple(mism[0])]}"
    ok = rst == 0
    if full:
        rb = ref["b"]
        rv = np.diagonal(ref["Var"], axis1=-2, axis2=-1)
    else:
        rb = ref["b"][..., -1]
        rv = ref["Var"][..., -1, -1]
    if not ok.any():
        return 0.0, 0.0
    bad = ~ok
    assert np.isnan(b[bad]).all() and np.isnan(v[bad]).all()
    eb = np.max(np.abs(b[ok] - rb[ok]) / np.sqrt(rv[ok]))
    ev = np.max(np.abs(v[ok] - rv[ok]) / rv[ok])
    return float(eb), float(ev)
