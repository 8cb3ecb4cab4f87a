"""Serving-loop workload on host-only handles: the KV-memory
metrics are exact chunk counts, checked against the paper's chunk arithmetic
(288 shared vs 1280 monolithic chunks for n_p = n_s = 2048,
n_c = 512, b = 32, c = 64; "reduced by 70%-90%") and against the
prefix-tree replay oracle C3 (oracle/tree_model.py) driven by the same op
stream."""
import pytest

from oracle.tree_model import TreeModel
from paper_2402_15220_b200 import ChunkAttention
from paper_2402_15220_b200.serving import ServingLoop, poisson_trace


def _loop(prefix_match, b_max=32, max_chunks=4096):
    ca = ChunkAttention(4, 64, 64, max_chunks, 64, 4096, prefix_match=prefix_match, device=None)
    return ServingLoop(ca, b_max)


def test_burst_peak_chunks_match_chunk_arithmetic():
    """lambda -> inf burst of b_max identical-prompt requests (Table-5 shape):
    peak = 32 shared + 32 x 8 private = 288 chunks vs 32 x 40 = 1280."""
    trace = poisson_trace(0, 32, 0.0, 2048, 2048, 512)
    shared = _loop(True).run(trace, "shared")
    mono = _loop(False).run(trace, "monolithic")
    assert shared.peak_batch == mono.peak_batch == 32
    assert shared.peak_kv_chunks == 32 + 32 * 8 == 288
    assert mono.peak_kv_chunks == 32 * 40 == 1280
    assert shared.peak_kv_chunks / mono.peak_kv_chunks <= 0.30
    assert shared.prefill_tokens_computed == 2048 and mono.prefill_tokens_computed == 32 * 2048
    assert shared.prefill_tokens_matched + shared.prefill_tokens_computed == 32 * 2048  # accounting conservation


def test_no_sharing_gives_equal_memory():
    trace = poisson_trace(1, 8, 0.0, 256, 0, 16)
    a = _loop(True).run(trace, "shared")
    b = _loop(False).run(trace, "monolithic")
    assert a.peak_kv_chunks == b.peak_kv_chunks and a.peak_kv_bytes == b.peak_kv_bytes


@pytest.mark.parametrize("rps", [200.0, 2000.0])
def test_poisson_run_matches_tree_oracle_and_is_deterministic(rps):
    """Replay the loop's tree ops through C3: the live chunk count after every
    iteration's peak equals the oracle's; two runs with one seed are identical."""
    trace = poisson_trace(2, 24, rps, 320, 192, 40)
    m1 = _loop(True, b_max=8).run(trace, "shared")
    m2 = _loop(True, b_max=8).run(trace, "shared")
    assert m1 == m2
    assert m1.requests == 24 and m1.iterations >= 40 and m1.peak_batch <= 8
    # oracle: same admission order -> peak chunk count from the replay model
    tm = TreeModel(64, 4096)
    peak = 0
    running = {}
    pending = sorted(trace, key=lambda r: r.arrival_s)
    clock = 0.0
    step = 0
    import synth
    while pending or running:
        if not running and pending and pending[0].arrival_s * 1e3 > clock:
            clock = pending[0].arrival_s * 1e3
        while pending and pending[0].arrival_s * 1e3 <= clock and len(running) < 8:
            r = pending.pop(0)
            sid, _, _ = tm.add_sequence(r.prompt)
            running[sid] = [r, 0]
        sids = list(running)
        tm.append(sids, [int(synth.hash_py(0, synth.TAG_DECODE, s, running[s][1]) % 31999 + 1) for s in sids])
        for s in sids:
            running[s][1] += 1
        peak = max(peak, tm.memory_stats()[0])
        clock += 1.0
        step += 1
        for s in list(running):
            if running[s][1] >= running[s][0].n_c:
                del running[s]
                tm.remove_sequence(s)
    assert m1.peak_kv_chunks == peak
    assert m1.iterations == step
