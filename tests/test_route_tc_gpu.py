"""Tensor-core router (be_qnet_route_tc, route_tc.cu) against the fp64 router
(be_qnet_route_f64) and the reference-recorded decisions.

Bar: every action identical to the fp64 router's (the tcgen05 result is only
used where its error bound certifies the decision; the rest is re-evaluated
with the fp64 router's exact arithmetic); Q values within 1e-5 relative
(+1e-6 absolute) of fp64 — the north star's fp32 tolerance."""
import numpy as np
import pytest
import torch

import goldens
from paper_2401_07886_b200 import QNetwork, TensorCoreRouter, route
from paper_2401_07886_b200._lib import InvalidParameterError

pytestmark = pytest.mark.gpu


def random_states(rng, B, T, M, scales=(128.0, 32.0, 8.0, 16.0), max_rate=60.0):
    x = np.zeros((B, T + M + 1))
    x[np.arange(B), rng.integers(0, T, B)] = 1.0
    for m in range(M):
        x[:, T + m] = rng.integers(0, 3 * int(scales[m % len(scales)]), B) / scales[m % len(scales)]
    x[:, -1] = rng.uniform(0.0, max_rate, B) / 48.0
    return x


def compare(net, x, cuda, eps=0.0, seed=0, counter=0):
    xt = torch.as_tensor(x, device=cuda)
    q64, a64 = route(net, xt, eps, seed, counter)
    r = TensorCoreRouter(net, cuda)
    q32, a32 = r(xt, eps, seed, counter)
    torch.cuda.synchronize()
    assert torch.equal(a32, a64), f"{int((a32 != a64).sum())} actions differ"
    q64n, q32n = q64.cpu().numpy(), q32.cpu().double().numpy()
    err = np.abs(q32n - q64n)
    assert np.all(err <= 1e-5 * np.abs(q64n) + 1e-6), f"max Q error {err.max():.3g}"
    return r.fallback_stats()


@pytest.mark.parametrize("seed", range(4))
def test_random_nets_match_fp64_router(cuda, seed):
    rng = np.random.default_rng(seed)
    T, M = 4, 3
    net = QNetwork.init_random(T, M, 256, rng)
    net.b1 = rng.normal(0, 0.1, 256)  # non-zero biases exercise the bias input
    net.b2 = rng.normal(0, 0.1, M)
    n, fb = compare(net, random_states(rng, 100_003, T, M), cuda)
    assert n == 100_003 and fb < n


@pytest.mark.parametrize("M,spread", [(3, 1e-3), (3, 1e-5), (4, 1e-4), (2, 1e-6)])
def test_correlated_columns_near_ties(cuda, M, spread):
    """W2 columns that differ by `spread` (as trained Q heads do, only more so):
    the margins are tiny, the per-action error bound would certify almost nothing,
    and the pairwise bound (layer-1 error through the column differences) decides
    most states on the tensor cores. Every action must still equal fp64's."""
    rng = np.random.default_rng(int(spread * 1e7) + M)
    T = 4
    net = QNetwork.init_random(T, M, 256, rng)
    base = rng.normal(0, 0.1, 256)
    net.w2 = base[:, None] + spread * rng.normal(0, 0.1, (256, M))
    net.b1 = rng.normal(0, 0.1, 256)
    net.b2 = spread * rng.normal(0, 0.1, M)
    n, fb = compare(net, random_states(rng, 60_001, T, M), cuda)
    assert n == 60_001
    if spread >= 1e-3:
        assert fb < n // 2, f"pairwise bound certified only {n - fb} of {n}"


def test_trained_policy_states_match_fp64_and_reference(cuda):
    """States the reference visited with its trained policy: actions equal the
    fp64 router's and the reference's own decisions (goldens carry the fp64
    reference top-2 margin; all exceed 1e-9)."""
    for name in ("unpredictable-1_trained", "unpredictable-2_trained", "stable_trained",
                 "single-task-0_trained", "cfg1_4_trained_t1"):
        g = goldens.load(name)
        m = g["meta"]
        T = len(m["reward"]["tasks"])
        sc = np.array(m["enc"]["batch_scales"])
        n = len(g["arrival"])
        x = np.zeros((n, T + len(sc) + 1))
        x[np.arange(n), g["task"]] = 1.0
        x[:, T:T + len(sc)] = g["obs"] / sc
        x[:, -1] = g["rate"] / m["enc"]["rate_scale"]
        net = QNetwork.from_any(goldens.net_for(m))
        compare(net, x, cuda)
        _, a = TensorCoreRouter(net, cuda)(torch.as_tensor(x, device=cuda))
        assert np.array_equal(a.cpu().numpy(), g["tier"]), name


def test_exact_ties_fall_back_and_take_the_first_maximum(cuda):
    rng = np.random.default_rng(5)
    net = QNetwork.init_random(4, 3, 256, rng)
    net.w2[:, 2] = net.w2[:, 1]
    net.b2[:] = [0.0, 10.0, 10.0]  # actions 1 and 2 tie exactly and dominate
    x = random_states(rng, 5000, 4, 3)
    n, fb = compare(net, x, cuda)
    assert fb == n
    _, a = route(net, torch.as_tensor(x, device=cuda))
    assert not bool((a == 2).any())


def test_epsilon_greedy_matches_fp64_router(cuda):
    rng = np.random.default_rng(9)
    net = QNetwork.init_random(4, 3, 256, rng)
    compare(net, random_states(rng, 20_000, 4, 3), cuda, eps=0.3, seed=77, counter=12)


@pytest.mark.parametrize("B", [1, 127, 128, 129, 1000, 33_333])
def test_partial_tiles(cuda, B):
    rng = np.random.default_rng(B)
    net = QNetwork.init_random(4, 3, 256, rng)
    compare(net, random_states(rng, B, 4, 3), cuda)


@pytest.mark.parametrize("T,M,H", [(1, 3, 256), (4, 1, 64), (2, 2, 32), (4, 4, 128), (8, 4, 96), (10, 3, 256)])
def test_shapes(cuda, T, M, H):
    rng = np.random.default_rng(T * 100 + M * 10 + H)
    net = QNetwork.init_random(T, M, H, rng)
    net.b1 = rng.normal(0, 0.05, H)
    compare(net, random_states(rng, 4096, T, M), cuda)


def test_unsupported_shapes_raise(cuda):
    with pytest.raises(InvalidParameterError):
        TensorCoreRouter(QNetwork.init_random(4, 5, 256, np.random.default_rng(0)), cuda)
    with pytest.raises(InvalidParameterError):
        TensorCoreRouter(QNetwork.init_random(4, 3, 512, np.random.default_rng(0)), cuda)
