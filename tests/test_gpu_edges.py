"""Edge cases of the parameters the paper fixes (gamma in (0, 1], tau in
[0, 1]; P:451 minimum budget) and of the head layout, against the oracle."""
import numpy as np
import pytest

import oracle
from synth import gen
from synth.configs import Workload
from tests import parity
from tests.test_gpu_parity import (MAX_ABS, MEAN_ABS, _check_attn_stagewise, _check_plan,
                                   _check_select_stagewise, _oracle_plans)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fp():
    import paper_2502_20766_b200 as m
    m.load_library()
    return m


def _stagewise(fp, w, **kw):
    q, k, v = gen.make_layer_bits(w)
    Q, K, V = parity.oracle_inputs(q, k, v)
    res = parity.run_gpu(fp, w, q, k, v, **kw)
    return res, Q, K, V


@pytest.mark.parametrize("gamma", [0.02, 0.3])
def test_small_gamma(fp, gamma):
    """gamma far below the defaults: very few lines / blocks reach the mass
    (K = 1 when the top element alone covers gamma T); forced blocks remain."""
    w = Workload("small-gamma", 4, 1, 2048, gamma, 0.1, 0, 201)
    res, Q, K, V = _stagewise(fp, w)
    _check_plan(w, res, _oracle_plans(w, Q, K))
    _check_select_stagewise(w, res, gamma, 0)
    _check_attn_stagewise(w, res, Q, K, V)
    nb = 16
    assert all(s["nnz_blocks"] >= 2 * nb - 1 for s in res["stats"])


@pytest.mark.parametrize("tau,want", [(0.0, oracle.VS), (1.0, oracle.QA)])
def test_tau_extremes(fp, tau, want):
    """tau = 0: D < 0 never holds -> every head Vertical-Slash; tau = 1: D < 1
    for any two distributions with a common support -> every head Query-Aware
    (readings A1 / A14)."""
    w = Workload("tau-ext", 8, 2, 2048, 0.9, tau, 0, 203)
    res, Q, K, V = _stagewise(fp, w)
    assert np.all(res["pattern"] == want), res["jsd"]
    _check_plan(w, res, _oracle_plans(w, Q, K))
    _check_select_stagewise(w, res, 0.9, 0)
    _check_attn_stagewise(w, res, Q, K, V, qblocks=[0, 5, 15])


def test_min_budget_covers_everything(fp):
    """a minimum budget of n tokens makes every row dense (clamped to qb + 1,
    A12): the sparse kernel then runs exactly the dense kernel's block lists, so
    the outputs are bitwise equal."""
    w = Workload("mb-all", 4, 1, 2048, 0.9, 0.1, 2048, 205)
    q, k, v = gen.make_layer_bits(w)
    res = parity.run_gpu(fp, w, q, k, v, dense=True)
    nb = 16
    assert np.all(res["row_ptr"][:, -1] == nb * (nb + 1) // 2)
    assert np.array_equal(res["out"], res["dense"])


def test_mha_group_one(fp):
    """GQA group size 1 (as many KV heads as Q heads), ragged n."""
    w = Workload("mha", 4, 4, 1500, 0.9, 0.1, 0, 207)
    res, Q, K, V = _stagewise(fp, w)
    _check_plan(w, res, _oracle_plans(w, Q, K))
    _check_select_stagewise(w, res, 0.9, 0)
    _check_attn_stagewise(w, res, Q, K, V)


def test_odd_block_count_pairs(fp):
    """an odd number of q-blocks (the last v8 pair has no second row), with the
    dense kernel on the same shape vs the oracle."""
    w = Workload("odd-nb", 4, 2, 128 * 7, 0.95, 0.1, 512, 209)
    q, k, v = gen.make_layer_bits(w)
    Q, K, V = parity.oracle_inputs(q, k, v)
    res = parity.run_gpu(fp, w, q, k, v, dense=True)
    _check_select_stagewise(w, res, w.gamma, w.min_budget)
    _check_attn_stagewise(w, res, Q, K, V)
    for h in range(w.heads):
        ref = oracle.dense_causal_attention(Q[h], K[h // 2], V[h // 2])
        d = np.abs(res["dense"][h] - ref)
        assert d.max() <= MAX_ABS and d.mean() <= MEAN_ABS
