"""The CP-ALS partial contraction (the MTTKRP GEMM of cp_als.cpp:296-303, as
the device's dimension tree forms it: T = Y x_mode F over all restarts) on
the int8 tensor cores with exact digit splitting (csrc/ozaki.cu), against an
extended-precision (np.longdouble) product of the same fp64 operands.

Bound checked: |T_dev - T_exact| <= tol * (|Y| x_mode |F|) elementwise, the
condition-free error measure of a dot product; tol = 4e-15 (the digit split
keeps 55 bits of every row's / column's largest value, so its error is a few
units of 2^-53 of the scale product; the DMMA GEMM's rounding error grows
with K and is checked at K * 2^-53)."""
import numpy as np
import pytest

import paper_1807_01350_b200 as ob

pytestmark = pytest.mark.gpu

TOL_OZAKI = 4e-15


def _exact_t(y, f, mode):
    """T[p][m, s R + r] in long double; m = the two remaining indices, first fastest."""
    p, q = y.shape[0], y.shape[1]
    s, r = f.shape[1], f.shape[4]
    out = np.zeros((p, q * q, s * r), dtype=np.longdouble)
    absout = np.zeros((p, q * q, s * r), dtype=np.longdouble)
    for i in range(p):
        yl = y[i].astype(np.longdouble)
        fc = np.concatenate([f[i, j, mode] for j in range(s)], axis=1).astype(np.longdouble)  # q x sR
        # A(m, k): the unfolding with the contracted mode as columns
        if mode == 2:
            a = yl.reshape(q * q, q, order="F")                      # rows i + Q j
        elif mode == 1:
            a = np.transpose(yl, (0, 2, 1)).reshape(q * q, q, order="F")  # rows i + Q k
        else:
            a = np.transpose(yl, (1, 2, 0)).reshape(q * q, q, order="F")  # rows j + Q k
        out[i] = a @ fc
        absout[i] = np.abs(a) @ np.abs(fc)
    return out, absout


def _scheme_bound(y, f, mode):
    """max|a_m| sum|b_n| + sum|a_m| max|b_n| for every (m, n) (long double)."""
    p, q = y.shape[0], y.shape[1]
    s = f.shape[1]
    out = []
    for i in range(p):
        yl = np.abs(y[i].astype(np.longdouble))
        if mode == 2:
            a = yl.reshape(q * q, q, order="F")
        elif mode == 1:
            a = np.transpose(yl, (0, 2, 1)).reshape(q * q, q, order="F")
        else:
            a = np.transpose(yl, (1, 2, 0)).reshape(q * q, q, order="F")
        fc = np.abs(np.concatenate([f[i, j, mode] for j in range(s)], axis=1).astype(np.longdouble))
        out.append(np.outer(a.max(axis=1), fc.sum(axis=0)) + np.outer(a.sum(axis=1), fc.max(axis=0)))
    return np.stack(out)


def _factors(rng, p, s, q, r, kind="unit"):
    f = rng.standard_normal((p, s, 3, q, r))
    if kind == "unit":
        f /= np.linalg.norm(f, axis=3, keepdims=True)
    return f


@pytest.mark.parametrize("q,s,r", [(20, 3, 5), (50, 2, 10), (64, 3, 20), (100, 1, 7), (128, 1, 32),
                                   (128, 3, 32), (100, 3, 30), (40, 5, 30)])
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_tgemm_digit_split_vs_exact(q, s, r, mode):
    rng = np.random.default_rng(1000 * q + 10 * r + mode)
    p = 2
    y = rng.standard_normal((p, q, q, q))
    y[1] = np.abs(y[1]) * 1e3 + 5.0  # positive, offset summaries (the streamed Y look like this)
    f = _factors(rng, p, s, q, r)
    t = ob.als_tgemm(y, f, mode, engine=1)
    ex, ab = _exact_t(y, f, mode)
    err = float(np.max(np.abs(t.astype(np.longdouble) - ex) / ab))
    t0 = ob.als_tgemm(y, f, mode, engine=0)
    err0 = float(np.max(np.abs(t0.astype(np.longdouble) - ex) / ab))
    print("q=%d s=%d r=%d mode=%d: digit split %.2e, DMMA %.2e" % (q, s, r, mode, err, err0))
    assert err <= TOL_OZAKI, err
    assert err0 <= q * 2.0 ** -53, err0


def test_tgemm_digit_split_dynamic_range_and_zeros():
    """Rows spanning 1e-120 .. 1e120, exact zeros, tiny columns.  The digit
    split is exact to 2^-55 of each row's (column's) largest value, so its
    error bound is the scheme's own: |err| <= tol (max|a| sum|b| + sum|a| max|b|)
    per dot product (an entry far below its row's largest is represented
    only to that absolute precision; the summaries and unit-column factors of
    CP-ALS have a narrow range within a row, where this is the bound above)."""
    rng = np.random.default_rng(7)
    p, q, s, r = 1, 32, 2, 6
    y = rng.standard_normal((p, q, q, q))
    y[0, :, :, 3] *= 1e120
    y[0, :, 5, :] *= 1e-120
    y[0, 7] = 0.0
    f = _factors(rng, p, s, q, r)
    f[0, 1, :, :, 2] *= 1e-60  # (every product stays a normal fp64 number)
    f[0, 0, :, :, 4] = 0.0
    for mode in range(3):
        t = ob.als_tgemm(y, f, mode, engine=1)
        ex, ab = _exact_t(y, f, mode)
        nz = ab > 0
        assert np.all(t[~nz] == 0.0)
        bound = _scheme_bound(y, f, mode)
        err = float(np.max(np.abs(t.astype(np.longdouble)[nz] - ex[nz]) / bound[nz]))
        assert err <= TOL_OZAKI, (mode, err)


def test_tgemm_digit_split_nonfinite_propagates():
    """A non-finite summary entry makes the outputs of its row NaN (the DMMA
    GEMM propagates it the same way), so the ALS non-finite checks fire."""
    rng = np.random.default_rng(3)
    p, q, s, r = 1, 16, 1, 4
    y = rng.standard_normal((p, q, q, q))
    y[0, 2, 3, 4] = np.nan
    f = _factors(rng, p, s, q, r)
    for mode in range(3):
        t = ob.als_tgemm(y, f, mode, engine=1)
        t0 = ob.als_tgemm(y, f, mode, engine=0)
        assert np.array_equal(np.isnan(t), np.isnan(t0)), mode
        assert np.isnan(t).any()
    f[0, 0, 1, 5, 2] = np.inf
    t = ob.als_tgemm(y, f, 1, engine=1)
    assert np.isnan(t[0, :, 2]).all()


@pytest.mark.parametrize("engine", ["i8", "dmma"])
def test_cp_als_sweeps_engines(monkeypatch, engine):
    """The batched CP-ALS sweeps' T-GEMMs go through the int8 tcgen05 kernel
    by default (path counter; OCTEN_ALS_TGEMM=dmma selects the DMMA GEMM),
    and either result matches the oracle restatement."""
    monkeypatch.setenv("OCTEN_ALS_TGEMM", engine)
    from oracle import octen_oracle as O
    from oracle import rng as R

    s = R.Substream(5)
    q, rank = 24, 4
    truth = O.KruskalModel([s.fill_uniform(q, rank) for _ in range(3)], np.ones(rank))
    y = O.reconstruct_fast(truth)
    y = y + 0.01 * np.random.default_rng(5).standard_normal(y.shape) * np.sqrt(np.mean(y * y))
    cfg = ob.AlsConfig(rank=rank, max_iters=40, rel_tol=1e-10, n_restarts=2)
    c0 = ob.kernel_counts()
    models, fits, its = ob.cp_als_batched([y, 2.0 * y], cfg, [11, 12])
    c1 = ob.kernel_counts()
    if engine == "i8":
        assert c1["tcgen05_als"] > c0["tcgen05_als"]
    else:
        assert c1["tcgen05_als"] == c0["tcgen05_als"]
    for yy, m, sd, fit in zip([y, 2.0 * y], models, [11, 12], fits):
        ref = O.cp_als(yy, O.AlsConfig(rank, 40, 1e-10, 2, sd))
        cg = min(O.congruence(O.KruskalModel(m.factors, m.lambda_), ref.model))
        print("fit %.12f oracle %.12f congruence %.12f" % (fit, ref.fit, cg))
        assert abs(fit - ref.fit) < 1e-8
        assert cg > 1 - 1e-7
