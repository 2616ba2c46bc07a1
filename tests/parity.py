"""Comparison rules shared by the GPU parity tests.

These encode the north star's bars: floats max-abs <= 1e-3; quantised symbols equal
except where the oracle's pre-round value is within 1e-4 of a .5 tie, with at most 1e-4
of elements differing; CDF indexes equal except within 1e-4 (relative) of a table
boundary, same cap; bitstreams bit-exact.
"""
import numpy as np

FLOAT_TOL = 1e-3
TIE_EPS = 1e-4
CAP = 1e-4


def check_float(got, ref, tol=FLOAT_TOL, what=""):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    assert np.all(np.isfinite(got)), what
    err = np.abs(got - ref)
    worst = float(err.max()) if err.size else 0.0
    assert worst <= tol, f"{what}: max-abs {worst:.3e} > {tol} at {np.unravel_index(err.argmax(), err.shape)}"
    return worst


def check_symbols(got, ref, v_oracle, what=""):
    """got/ref int symbols; v_oracle = the oracle's fp32 pre-round value (y - mu)."""
    got = np.asarray(got).astype(np.int32)
    ref = np.asarray(ref).astype(np.int32)
    bad = got != ref
    n = int(bad.sum())
    if n:
        v = np.asarray(v_oracle, np.float64)[bad]
        frac = np.abs(np.abs(v) - np.floor(np.abs(v)) - 0.5)
        assert np.all(frac < TIE_EPS), f"{what}: {n} symbol mismatches, not all at .5 ties"
        assert np.all(np.abs(got[bad] - ref[bad]) == 1), what
        assert n <= max(1, CAP * got.size), f"{what}: {n} mismatches > cap"
    return n


def check_indexes(got, ref, sigma_oracle, table, what=""):
    got = np.asarray(got).astype(np.int32)
    ref = np.asarray(ref).astype(np.int32)
    bad = got != ref
    n = int(bad.sum())
    if n:
        s = np.maximum(np.asarray(sigma_oracle, np.float64)[bad], 0.11)
        j = np.minimum(got[bad], ref[bad])            # boundary between index j and j+1 is table_j
        assert np.all(np.abs(got[bad] - ref[bad]) == 1), what
        t = np.asarray(table, np.float64)[j]
        assert np.all(np.abs(s - t) <= TIE_EPS * t), f"{what}: {n} index mismatches away from a boundary"
        assert n <= max(1, CAP * got.size), f"{what}: {n} mismatches > cap"
    return n
