"""Host-side logic of the drop-in API that runs without a GPU: parameter
initialisation (bit-identical to the reference), validation and errors."""
import glob
import os

import numpy as np
import pytest

import paper_2602_08810_b200 as lrx
from tests.conftest import GOLDEN


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "layer_*.npz"))),
                         ids=lambda p: os.path.basename(p)[6:-4])
def test_parameter_init_matches_reference(path):
    z = np.load(path)
    n = int(z["d_state"])
    layer = lrx.make_layer(str(z["kind"]), int(z["d_model"]), None if n < 0 else n,
                           str(z["scheme"]) or None, asynchronous="deltas" in z.files,
                           dtype=str(z["dtype"]), seed=int(z["seed"]), device="cpu")
    params = layer.parameters()
    want = {k[6:]: z[k] for k in z.files if k.startswith("param:")}
    assert list(params) == list(want)  # same keys, same order
    for k, v in want.items():
        np.testing.assert_array_equal(params[k].numpy(), v, err_msg=k)


def test_registry_and_errors():
    with pytest.raises(lrx.UnknownLayer):
        lrx.make_layer("s7", 4, device="cpu")
    with pytest.raises(ValueError):
        lrx.make_layer("s5", 4, 5, device="cpu")  # odd d_state
    with pytest.raises(ValueError):
        lrx.make_layer("s4d", 4, discretization="euler", device="cpu")
    with pytest.raises(ValueError):
        lrx.make_layer("lru", 4, dtype="bf16", device="cpu")
    with pytest.warns(UserWarning):
        lrx.make_layer("lru", 4, discretization="zoh", device="cpu")
    layer = lrx.make_layer("s6", 4, dtype="bf16", device="cpu")
    assert layer.parameters()["a_log"].dtype.is_floating_point


def test_cpu_layer_refuses_to_compute():
    layer = lrx.make_layer("rglru", 4, device="cpu")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        layer.forward(np.zeros((1, 3, 4)))


def test_plan_chunks_and_combine_host():
    assert lrx.plan_chunks(513, 2) == [(0, 257), (257, 513)]
    a, b = lrx.combine((np.array(0.5), np.array(1.0)), (np.array(0.5), np.array(1.0)))
    assert a == 0.25 and b == 1.5
    with pytest.raises(lrx.ShapeError):
        lrx.combine((np.zeros(3), np.zeros(3)), (np.zeros(4), np.zeros(4)))


def test_host_numerics():
    x = np.array([-100.0, 0.0, 40.0, 60.0])
    np.testing.assert_allclose(lrx.softplus(x), [0.0, np.log(2), 40.0, 60.0], atol=1e-15)
    np.testing.assert_allclose(lrx.sigmoid(np.array([-800.0, 0.0, 800.0])), [0.0, 0.5, 1.0])
    assert lrx.real_dtype("f32") == np.float32


def test_init_invariants():
    """The reference's initialisation invariants (test_layers.py:128-176),
    checked on the drop-in layers' parameters (CPU, no compute)."""
    m, n = 8, 6
    s4d = lrx.make_layer("s4d", m, n, device="cpu")
    lam_re = -np.exp(s4d.parameters()["lambda_re_log"].numpy())
    np.testing.assert_allclose(lam_re, -0.5)  # S4D-Lin: lambda = -1/2 + i pi n
    np.testing.assert_allclose(s4d.parameters()["lambda_im"].numpy(), np.pi * np.arange(n)[None, :].repeat(m, 0))
    lru = lrx.make_layer("lru", m, n, device="cpu", r_min=0.9, r_max=0.999, max_phase=np.pi / 10)
    p = {k: v.numpy() for k, v in lru.parameters().items()}
    mag = np.exp(-np.exp(p["nu_log"]))
    assert np.all((mag >= 0.9 - 1e-12) & (mag <= 0.999 + 1e-12))  # the LRU ring
    phase = np.exp(p["theta_log"])
    assert np.all((phase > 0) & (phase <= np.pi / 10 + 1e-12))
    np.testing.assert_allclose(np.exp(p["gamma_log"]), np.sqrt(1 - mag ** 2), rtol=1e-12)
    s6 = lrx.make_layer("s6", m, n, device="cpu")
    q = {k: v.numpy() for k, v in s6.parameters().items()}
    np.testing.assert_allclose(-np.exp(q["a_log"]), -np.arange(1, n + 1)[None, :].repeat(m, 0))  # a = -(n+1)
    dt = lrx.softplus(q["b_delta"])
    assert np.all((dt >= 1e-3 - 1e-12) & (dt <= 1e-1 + 1e-12))
    rg = lrx.make_layer("rglru", m, device="cpu")
    a = lrx.sigmoid(rg.parameters()["lambda_param"].numpy())
    assert np.all((a >= 0.9 - 1e-12) & (a <= 0.999 + 1e-12))


def test_numerics_helpers():
    """as_tensor / complex_exp / ComplexPair / allocation_count (reference
    numerics.py:67-175)."""
    assert lrx.as_tensor([1, 2]).dtype == np.float64
    assert lrx.as_tensor(np.ones(2, np.complex64)).dtype == np.complex64
    assert lrx.as_tensor([1.0], dtype="f32").dtype == np.float32
    with pytest.raises(ValueError):
        lrx.as_tensor([1], dtype=np.int32)
    z = np.array([0.3 + 1.2j, -2.0 + 0.1j])
    np.testing.assert_allclose(lrx.complex_exp(z), np.exp(z), rtol=1e-15)
    re, im = lrx.complex_exp(z.real, z.imag)
    np.testing.assert_allclose(re + 1j * im, np.exp(z), rtol=1e-15)
    with pytest.raises(lrx.ShapeError):
        lrx.complex_exp(np.zeros(2), np.zeros(3))
    p = lrx.ComplexPair.from_complex(z.astype(np.complex64))
    assert p.shape == (2,) and p.to_complex().dtype == np.complex64
    np.testing.assert_allclose(p.to_complex(), z.astype(np.complex64))
    with pytest.raises(lrx.ShapeError):
        lrx.ComplexPair(np.zeros(2), np.zeros(3))
    n0 = lrx.allocation_count()
    lrx.alloc((3,), np.float32)
    assert lrx.allocation_count() == n0 + 1
