"""Pin the bytes/flops model to Table 1."""
import os

from paper_2402_15220_b200.roofline import StepShape, table1_self_attention

GOLD = os.path.join(os.path.dirname(__file__), "golden", "table1_roofline.txt")


def test_table1_flops_mops_within_5pct():
    rows = []
    with open(GOLD) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                b, fl, mo = line.split()
                rows.append((int(b), float(fl) * 1e6, float(mo) * 1e6))
    assert len(rows) == 3
    for b, fl, mo in rows:
        f, m = table1_self_attention(b)
        assert abs(f - fl) / fl < 0.05 and abs(m - mo) / mo < 0.05, (b, f, fl, m, mo)
        assert abs(f - fl) / fl < 0.01                  # 4bhnd is the printed FLOPs to <1%


def test_step_shape_monolithic_equals_table1():
    """No sharing (every token private) reproduces Table 1's MOPs exactly."""
    b, n = 32, 2048
    s = StepShape(b=b, h=32, d=128, c=64, elem=2, out_elem=2, shared_chunks=0, shared_rows=0, q_rows_cf=0,
                  private_tokens=b * n)
    f, m = table1_self_attention(b)
    assert s.seq_first_bytes() == m
    assert s.seq_first_flops() == f


def test_config2_bytes():
    """Config 2 (b=32, h=32, d=128, fp16, n_s=2048) at p private tokens:
    16 KiB of K+V per token, (2048 + 32 p) distinct tokens, + q and o."""
    for p in (1, 65):
        s = StepShape(b=32, h=32, d=128, c=64, elem=2, out_elem=2, shared_chunks=32, shared_rows=32 * 32,
                      q_rows_cf=32, private_tokens=32 * p)
        assert s.unique_bytes() == 16384 * (2048 + 32 * p) + 32 * 32 * 128 * 2 * 2
        # per-kernel figures each include the query rows they read
        assert s.chunk_first_bytes() + s.seq_first_bytes() == s.unique_bytes() + 32 * 32 * 128 * 2
    assert abs(StepShape(32, 32, 128, 64, 2, 2, 32, 1024, 32, 32).unique_bytes() / 1e6 - 34.6) < 0.05
