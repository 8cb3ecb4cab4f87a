"""Pins for the shared seeded generator (synth/)."""
import torch

import synth


def test_hash_matches_pure_python():
    for keys in [(0,), (1, 2, 3), (7, 1, 99999, 2048), (0xFFFFFFFF, 5)]:
        assert int(synth.hash_keys(*keys)) == synth.hash_py(*keys)
    idx = torch.arange(1000)
    h = synth.hash_keys(3, 1, idx)
    for i in (0, 1, 17, 999):
        assert int(h[i]) == synth.hash_py(3, 1, i)


def test_values_exact_in_half_types():
    tok = synth.token_ids(0, synth.TAG_SYS, 0, 300)
    assert int(tok.min()) >= 1 and int(tok.max()) <= 31999
    k = synth.kv_values(0, synth.TID_K, tok, torch.arange(300), 2, 4, 64)
    assert k.shape == (300, 2, 4, 64)
    for dt in (torch.float16, torch.bfloat16, torch.float32):
        for a in (1.0, 8.0, 16.0):
            x = k * a
            assert torch.equal(x.to(dt).to(torch.float64), x)
    assert float(k.min()) >= -1.0 and float(k.max()) <= 127 / 128
    # roughly uniform byte: mean near -1/256, std near 0.577
    assert abs(float(k.mean())) < 0.02 and 0.5 < float(k.std()) < 0.65


def test_kv_depends_only_on_token_and_position():
    t = torch.tensor([5, 6, 5])
    p = torch.tensor([0, 1, 0])
    k = synth.kv_values(1, synth.TID_K, t, p, 1, 2, 8)
    assert torch.equal(k[0], k[2]) and not torch.equal(k[0], k[1])
    v = synth.kv_values(1, synth.TID_V, t, p, 1, 2, 8)
    assert not torch.equal(k, v)
    # head slice of a sharded rank equals the slice of the full tensor
    full = synth.kv_values(1, synth.TID_K, t, p, 1, 8, 8)
    part = synth.kv_values(1, synth.TID_K, t, p, 1, 2, 8, head_offset=4)
    assert torch.equal(full[:, :, 4:6], part)
