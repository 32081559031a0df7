"""Pin the oracle restatement (oracle/port.py + oracle/scan_loops.c) to the
reference: golden vectors produced by the real linrec (tests/golden/) and the
known-answer values of the reference's own test-suite."""
import glob
import os

import numpy as np
import pytest

from oracle import port
from tests.conftest import GOLDEN

LAYER_FILES = sorted(glob.glob(os.path.join(GOLDEN, "layer_*.npz")))


def _load(path):
    z = np.load(path, allow_pickle=False)
    return {k: z[k] for k in z.files}


def _case(rec):
    kind = str(rec["kind"])
    scheme = str(rec["scheme"]) or None
    n = int(rec["d_state"])
    params = {k[6:]: v for k, v in rec.items() if k.startswith("param:")}
    grads = {k[5:]: v for k, v in rec.items() if k.startswith("grad:")}
    return kind, scheme, (None if n < 0 else n), params, grads


@pytest.mark.parametrize("path", LAYER_FILES, ids=lambda p: os.path.basename(p)[6:-4])
def test_oracle_matches_reference_layer(path):
    rec = _load(path)
    kind, scheme, n, params, grads = _case(rec)
    dtype = str(rec["dtype"])
    # parameter initialisation replays the reference's Philox streams exactly
    mine = port.init_params(kind, int(rec["d_model"]), n, dtype=dtype, seed=int(rec["seed"]))
    assert set(mine) == set(params)
    for k in params:
        np.testing.assert_array_equal(mine[k], params[k], err_msg=k)
    layer = port.Layer(kind, mine, scheme, asynchronous="deltas" in rec)
    deltas = rec.get("deltas")
    tol = 1e-12 if dtype == "f64" else 2e-6
    for mode, workers in (("sequential", 1), ("parallel", 3)):
        y, saved = layer.forward(rec["u"], mode, workers, deltas)
        assert port.rel_err(y, rec["y"]) < tol, mode
        g, gu = layer.backward(saved, rec["gy"])
        assert set(g) == set(grads)
        assert port.rel_err(gu, rec["gu"]) < tol
        for k in grads:
            assert g[k].shape == grads[k].shape, k
            gtol = tol if dtype == "f64" else 1e-4
            assert port.rel_err(g[k], grads[k]) < gtol, (k, port.rel_err(g[k], grads[k]))
    if "y_par" in rec:
        assert port.rel_err(layer.forward(rec["u"], "parallel", 3, deltas)[0], rec["y_par"]) < tol


def test_oracle_naive_loops_agree_with_reference():
    for name in ("s4d_zoh", "s5_bilinear", "lru", "s6", "rglru", "s5_dirac_async"):
        rec = _load(os.path.join(GOLDEN, f"layer_{name}.npz"))
        kind, scheme, n, params, _ = _case(rec)
        y = port.naive_forward(kind, params, rec["u"], scheme, rec.get("deltas"))
        assert port.rel_err(y, rec["y"]) < 1e-11, name


@pytest.mark.parametrize("key", ["real_const", "real_var", "cplx_const", "cplx_var"])
def test_oracle_scan_ops_match_reference(key):
    z = np.load(os.path.join(GOLDEN, "scan_ops.npz"))
    a, b, x0 = z[key + ":a"], z[key + ":b"], z[key + ":x0"]
    # the C loops keep the reference's operation order: sequential is bit-exact
    np.testing.assert_array_equal(port.scan_sequential(a, b, x0), z[key + ":seq"])
    np.testing.assert_array_equal(port.scan_parallel(a, b, x0, workers=3), z[key + ":par3"])
    states = port.scan_sequential(a, b, x0)
    ga, gb, gx0 = port.scan_backward(a, states, x0, z[key + ":gx"])
    np.testing.assert_allclose(ga, z[key + ":ga"], rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(gb, z[key + ":gb"], rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(gx0, z[key + ":gx0"], rtol=1e-13, atol=1e-13)


# --- known-answer values from the reference test-suite ------------------------

def test_kat_unrolled_scan():  # test_scan.py:19-25
    np.testing.assert_array_equal(port.scan_sequential(np.array(0.5), np.ones(3)), [1.0, 1.5, 1.75])
    np.testing.assert_array_equal(port.scan_sequential(np.array(0.5), np.ones(3), x0=np.array(1.0)),
                                  [1.5, 1.75, 1.875])


def test_kat_combine_and_halving():  # test_scan.py:28-30, 112-117
    a, b = port.combine((np.array(0.5), np.array(1.0)), (np.array(0.5), np.array(1.0)))
    assert a == 0.25 and b == 1.5
    out = port.scan_sequential(np.array([0.5]), np.zeros((4, 1)), x0=np.array([16.0]))
    np.testing.assert_array_equal(out[:, 0], [8.0, 4.0, 2.0, 1.0])


def test_kat_plan_chunks():  # test_scan.py:60-67
    assert port.plan_chunks(100, 8) == [(0, 100)]
    assert port.plan_chunks(512, 2) == [(0, 256), (256, 512)]
    assert port.plan_chunks(513, 2) == [(0, 257), (257, 513)]


def test_kat_discretization():  # test_discretize.py:23-58
    A, DT = np.array([-1.0 + 0.0j]), np.array([0.1])
    ab, sc = port.scheme_factors("zoh", A, DT)
    assert ab[0] == pytest.approx(0.9048374180359595, abs=1e-15)
    assert sc[0] == pytest.approx(0.09516258196404048, abs=1e-15)
    ab, sc = port.scheme_factors("bilinear", A, DT)
    assert ab[0] == pytest.approx(0.95 / 1.05, abs=1e-15)
    assert sc[0] == pytest.approx(0.1 / 1.05, abs=1e-15)
    ab, sc = port.scheme_factors("dirac", A, DT)
    assert ab[0] == pytest.approx(np.exp(-0.1), abs=1e-15) and sc[0] == 1.0
    ab, sc = port.scheme_factors("zoh", np.array([0.0 + 0.0j, 1e-12 + 0.0j]), np.array([0.25]))
    np.testing.assert_allclose(sc, [0.25, 0.25], atol=1e-10)
    with pytest.raises(port.SingularBilinear):
        port.scheme_factors("bilinear", np.array([2.0 + 0.0j]), np.array([1.0]))


def test_kat_length_one_f32():  # test_scan.py:155-160
    out = port.scan_sequential(np.array([0.5], np.float32), np.array([[2.0]], np.float32))
    assert out.dtype == np.float32
    np.testing.assert_array_equal(out, [[2.0]])


def test_s6_layer_blocked_equals_layer():
    """The channel-blocked S6 oracle (used for full-length C3 rows) equals the
    unblocked layer restatement (layers.py:1051-1118)."""
    params = port.init_params("s6", 12, 4, dtype="f64", seed=3)
    u = port.Rng(4).normal((2, 37, 12))
    gy = port.Rng(5).normal((2, 37, 12))
    lay = port.Layer("s6", params)
    ry, saved = lay.forward(u)
    rg, rgu = lay.backward(saved, gy)
    y, g, gu, extra = port.s6_layer_blocked(params, u, gy, block=5)
    assert port.rel_err(y, ry) < 1e-13
    assert port.rel_err(gu, rgu) < 1e-13
    assert set(g) == set(rg)
    for k in rg:
        assert port.rel_err(g[k], rg[k]) < 1e-12, k
