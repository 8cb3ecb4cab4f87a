"""Pins of the prefill oracle (oracle/prefill.py, C4) against values fixed by
the mathematics, not by re-calling its own routine."""
import numpy as np

from oracle.attention import attend_heads_fp64, default_scale
from oracle.prefill import causal_prefill_fp64


def _rand(seed, n, h, d):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((n, h, d)), rng.standard_normal((n, h, d)), rng.standard_normal((n, h, d))


def test_matches_masked_softmax_matrix_form():
    """softmax(s Q K^T + M) V, M = -inf strictly above the diagonal (the whole
    causal attention matrix at once), per head."""
    n, h, d, f = 11, 3, 8, 4
    q, K, V = _rand(0, n, h, d)
    s = default_scale(d)
    got = causal_prefill_fp64(q[f:], K, V, f, s)
    for hh in range(h):
        S = s * q[:, hh] @ K[:, hh].T
        S = np.where(np.tril(np.ones((n, n), dtype=bool)), S, -np.inf)
        P = np.exp(S - S.max(axis=1, keepdims=True))
        P /= P.sum(axis=1, keepdims=True)
        ref = P @ V[:, hh]
        np.testing.assert_allclose(got[:, hh], ref[f:], rtol=1e-12, atol=1e-13)


def test_position_zero_returns_first_value():
    q, K, V = _rand(1, 5, 2, 4)
    got = causal_prefill_fp64(q, K, V, 0, 0.5)
    np.testing.assert_allclose(got[0], V[0], rtol=0, atol=1e-15)


def test_constant_values_give_constant_output():
    q, K, _ = _rand(2, 7, 2, 4)
    V = np.ones_like(K)
    np.testing.assert_allclose(causal_prefill_fp64(q[3:], K, V, 3, 0.3), 1.0, rtol=0, atol=1e-14)


def test_last_query_is_the_decode_output():
    """first_pos = n - 1: the single query sees the whole sequence (C1)."""
    n, h, d = 9, 2, 4
    q, K, V = _rand(3, n, h, d)
    got = causal_prefill_fp64(q[n - 1:], K, V, n - 1, 0.7)
    np.testing.assert_allclose(got[0], attend_heads_fp64(q[n - 1], K, V, 0.7), rtol=1e-14, atol=1e-15)


def test_future_tokens_do_not_leak():
    """Changing K/V after position p leaves out_p unchanged."""
    n, h, d = 8, 2, 4
    q, K, V = _rand(4, n, h, d)
    a = causal_prefill_fp64(q, K, V, 0, 0.5)
    K2, V2 = K.copy(), V.copy()
    K2[5:] += 100.0
    V2[5:] -= 50.0
    b = causal_prefill_fp64(q, K2, V2, 0, 0.5)
    np.testing.assert_array_equal(a[:5], b[:5])
    assert np.abs(a[5:] - b[5:]).max() > 1e-3
