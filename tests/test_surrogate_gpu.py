"""GPU surrogate network (paper_2109_05948_b200/surrogate.py + csrc/segsum.cu)
against the reference's own numpy `SurrogateNet` (tests/golden/surrogate.npz,
made by tests/golden/make_golden.py from `mc/surrogate.py`): predictions of the
freshly initialised net, one minibatch's gradients (vs the hand-written
`_backward`, :180-217), per-epoch losses and predictions after two online
training generations (`train_generation`, :258-304), final parameters.

Tolerances: float64 nets agree to summation-order rounding (rtol 1e-9 on
outputs, 1e-7 after 30 Adam steps); float32 ones to float32 rounding carried
through training (rtol 2e-3 on losses and predictions; parameters within 10
Adam steps each)."""

import io

import numpy as np
import pytest
import torch

from conftest import load_golden
from paper_2109_05948_b200 import _native as N
from paper_2109_05948_b200.init import random_col_assigns
from paper_2109_05948_b200.rng import TAG_TRAIN, Stream
from paper_2109_05948_b200.surrogate import SurrogateNet

pytestmark = pytest.mark.gpu
G = load_golden("surrogate")
CASES = [str(c) for c in G["cases"]]


def _targets(assigns):  # tests/golden/make_golden.py:surrogate_targets
    a = assigns.astype(np.float64)
    return 3.0 * (assigns == 0).sum(axis=1) + 0.5 * a[:, 0] - 0.25 * a[:, -1] + 10.0


def _setup(name):
    n, k, seed, f64, bn, B, epochs, bs, gens = (int(x) for x in G[name + "__params"])
    net = SurrogateNet(n, problem="col", arch="small", seed=seed, dtype=np.float64 if f64 else np.float32,
                       use_bn=bool(bn))
    assigns = random_col_assigns(n, k, B, seed + 100)
    test = random_col_assigns(n, k, 16, seed + 200)
    tol = dict(rtol=1e-9, atol=1e-11) if f64 else dict(rtol=2e-3, atol=2e-4)
    return net, assigns, test, k, seed, epochs, bs, gens, tol, f64


@pytest.mark.parametrize("name", CASES)
def test_initial_predictions(name):
    net, _, test, k, *_, tol, f64 = _setup(name)
    np.testing.assert_allclose(net.predict_assigns(test, k), G[name + "__pred0"], **tol)


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("path", ["ids", "dense"])
def test_minibatch_gradients(name, path):
    net, assigns, _, k, *_, tol, f64 = _setup(name)
    y = _targets(assigns[:8])
    yz = torch.tensor((y - y.mean()) / y.std(), dtype=net.tdtype, device="cuda")
    params = net._flat_params()
    for p in params:
        p.requires_grad_(True)
    if path == "ids":
        pred = net.forward_assigns(assigns[:8], k, mode="train", update_running=False)
    else:
        pred = net.forward(net.one_hot(assigns[:8], k), mode="train", keep_cache=True, update_running=False)
    err = pred - yz
    grads = net._param_grads(torch.mean(err * err))
    np.testing.assert_allclose(pred.detach().double().cpu().numpy(), G[name + "__train_pred"], **tol)
    gt = dict(rtol=1e-8, atol=1e-12) if f64 else dict(rtol=2e-3, atol=1e-5)
    for j, g in enumerate(grads):
        np.testing.assert_allclose(g.double().cpu().numpy(), G[name + f"__grad{j}"], err_msg=f"grad {j}", **gt)


@pytest.mark.parametrize("name", CASES)
def test_online_training(name):
    net, assigns, test, k, seed, epochs, bs, gens, tol, f64 = _setup(name)
    y = _targets(assigns)
    lt = dict(rtol=1e-7, atol=1e-10) if f64 else dict(rtol=2e-3, atol=2e-4)
    for t in range(gens):
        losses = net.train_generation(assigns, y + t, k, epochs, bs, Stream.derive(seed, TAG_TRAIN, t))
        np.testing.assert_allclose(losses, G[name + f"__g{t}_losses"], **lt)
        np.testing.assert_allclose(net.predict_assigns(test, k), G[name + f"__g{t}_pred"], **lt)
    assert net.adam_t == int(G[name + "__adam_t"])
    # float32: Adam's normalised step m / sqrt(v) turns rounding-level gradient
    # differences on near-zero gradients into +-lr steps, so each parameter is
    # within 10 steps (10 lr); losses and predictions above are the
    # statistical-parity check
    pt = lt if f64 else dict(rtol=0, atol=10 * net.lr)
    for i, layer in enumerate(net.layers):
        for nm in ("lam", "gam", "beta", "bn_scale", "bn_shift", "run_mean", "run_var"):
            got, ref = getattr(layer, nm).double().cpu().numpy(), G[name + f"__l{i}_{nm}"]
            np.testing.assert_allclose(got, ref, err_msg=f"l{i} {nm}", **pt)
    # checkpoint round trip (reference key layout)
    buf = io.BytesIO()
    net.save(buf)
    buf.seek(0)
    keys = set(np.load(io.BytesIO(buf.getvalue())).keys())
    assert {"meta", "l0_lam", "l0_run_var", "adam_m0", f"adam_v{5 * len(net.layers) - 1}"} <= keys
    net2 = SurrogateNet.load(buf)
    np.testing.assert_array_equal(net2.predict_assigns(test, k), net.predict_assigns(test, k))
    assert net2.adam_t == net.adam_t


def test_nonfinite_training_restores_snapshot():
    net = SurrogateNet(16, arch="small", seed=1, dtype=np.float32)
    a = random_col_assigns(16, 3, 12, 5)
    before = [p.clone() for p in net._flat_params()]
    losses = net.train_generation(a, np.full(12, np.inf), 3, 2, 4, Stream.derive(1, TAG_TRAIN, 0))
    assert losses == [] and net.train_events and net.adam_t == 0
    for p, q in zip(net._flat_params(), before):
        assert torch.equal(p, q)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_segsum_kernel_vs_one_hot_matmul(dtype):
    rs = np.random.default_rng(3)
    B, n, k, L = 37, 301, 19, 333
    a = torch.tensor(rs.integers(0, k, (B, n)), dtype=torch.int32, device="cuda")
    lam = torch.randn(n, L, dtype=dtype, device="cuda")
    x = torch.zeros(B, k, n, dtype=dtype, device="cuda").scatter_(1, a.long()[:, None, :], 1.0)
    z = torch.empty(B, k, L, dtype=dtype, device="cuda")
    es = 4 if dtype == torch.float32 else 8
    s = torch.cuda.current_stream().cuda_stream
    N.check(N.lib().mcb_segsum(es, 0, N.ptr(lam), N.ptr(a), B, n, k, L, N.ptr(z), s))
    ref = torch.matmul(x.double(), lam.double())
    tol = 1e-4 if dtype == torch.float32 else 1e-12
    torch.testing.assert_close(z.double(), ref, rtol=tol, atol=tol)
    dz = torch.randn(B, k, L, dtype=dtype, device="cuda")
    dl = torch.empty(n, L, dtype=dtype, device="cuda")
    N.check(N.lib().mcb_segsum(es, 1, N.ptr(dz), N.ptr(a), B, n, k, L, N.ptr(dl), s))
    torch.testing.assert_close(dl.double(), torch.einsum("bil,biL->lL", x.double(), dz.double()), rtol=tol, atol=tol)
    a[3, 7] = k  # out of range -> ValueError, like the reference's one-hot indexing
    with pytest.raises(ValueError):
        N.check(N.lib().mcb_segsum(es, 0, N.ptr(lam), N.ptr(a), B, n, k, L, N.ptr(z), s))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("use_bn", [True, False])
def test_fused_eval_path_matches_autograd_path(dtype, use_bn):
    """predict_assigns (colour-sorted segment sums + fused epilogues) equals
    the training-path forward in eval mode after some training (non-trivial
    running statistics)."""
    net = SurrogateNet(40, arch="small", seed=2, dtype=dtype, use_bn=use_bn)
    a = random_col_assigns(40, 7, 50, 4)
    net.train_generation(a, _targets(a), 7, 2, 8, Stream.derive(2, TAG_TRAIN, 0))
    test = random_col_assigns(40, 7, 33, 9)
    fast = net.predict_assigns(test, 7, chunk=16)
    with torch.no_grad():
        slow = net.forward_assigns(test, 7, mode="eval").double().cpu().numpy() * net.target_std + net.target_mean
    tol = 1e-10 if dtype == np.float64 else 1e-4
    np.testing.assert_allclose(fast, slow, rtol=tol, atol=tol)


def test_surrogate_api_edges():
    net = SurrogateNet(12, arch="small", seed=0)
    assert net.predict_assigns(np.zeros((0, 12), np.int32), 3).shape == (0,)
    with pytest.raises(ValueError):
        net.predict_assigns(np.zeros((2, 11), np.int32), 3)  # wrong vertex count
    with pytest.raises(ValueError):
        net.predict_assigns(np.full((2, 12), 3, np.int32), 3)  # colour id >= k
    with pytest.raises(ValueError):
        net.train_generation(np.zeros((0, 12), np.int32), np.zeros(0), 3, 1, 4, Stream.derive(0, TAG_TRAIN, 0))
    with pytest.raises(ValueError):
        net.forward(np.zeros((2, 3, 11)))
    # a single training example: std 0 -> 1 (`:266-268`), one minibatch of 1
    losses = net.train_generation(np.zeros((1, 12), np.int32), np.array([5.0]), 3, 2, 4,
                                  Stream.derive(0, TAG_TRAIN, 1))
    assert len(losses) == 2 and net.target_std == 1.0 and net.target_mean == 5.0


def test_tf32_option_is_close_and_off_by_default():
    """tf32=True (opt-in) runs the GEMMs on the tensor cores: predictions stay
    within TF32 rounding of the float32 net; the default leaves the global
    cuBLAS setting alone and computes in float32."""
    a = random_col_assigns(64, 6, 40, 3)
    test = random_col_assigns(64, 6, 30, 4)
    y = _targets(a)
    ref = SurrogateNet(64, arch="small", seed=5)
    fast = SurrogateNet(64, arch="small", seed=5, tf32=True)
    assert not ref.tf32 and fast.tf32
    before = torch.backends.cuda.matmul.allow_tf32
    ref.train_generation(a, y, 6, 2, 8, Stream.derive(5, TAG_TRAIN, 0))
    fast.train_generation(a, y, 6, 2, 8, Stream.derive(5, TAG_TRAIN, 0))
    p_ref, p_fast = ref.predict_assigns(test, 6), fast.predict_assigns(test, 6)
    assert torch.backends.cuda.matmul.allow_tf32 == before
    np.testing.assert_allclose(p_fast, p_ref, rtol=2e-2, atol=2e-2 * np.abs(p_ref).max())


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_graph_training_equals_eager(dtype):
    """CUDA-graph replays of the minibatch step (default) give exactly the
    eager step's parameters, moments, running statistics and losses --
    including a tail minibatch of another size and a second call that reuses
    the captured graphs."""
    a = random_col_assigns(30, 5, 45, 8)
    y = _targets(a)
    nets = [SurrogateNet(30, arch="small", seed=4, dtype=dtype) for _ in range(2)]
    for t in range(2):
        l0 = nets[0].train_generation(a, y + t, 5, 2, 8, Stream.derive(4, TAG_TRAIN, t), graphs=True)
        l1 = nets[1].train_generation(a, y + t, 5, 2, 8, Stream.derive(4, TAG_TRAIN, t), graphs=False)
        assert l0 == l1
    for p0, p1 in zip(nets[0]._flat_params() + nets[0].adam_m + nets[0].adam_v,
                      nets[1]._flat_params() + nets[1].adam_m + nets[1].adam_v):
        assert torch.equal(p0, p1)
    for l0, l1 in zip(nets[0].layers, nets[1].layers):
        assert torch.equal(l0.run_mean, l1.run_mean) and torch.equal(l0.run_var, l1.run_var)
    assert nets[0].adam_t == nets[1].adam_t == 2 * 2 * 6
