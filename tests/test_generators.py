import numpy as np

from paper_2605_26599_b200 import generators as G


def test_jump_ahead_equals_sequential():
    s = G.seed_for("sym-uniform", 77)
    seq, x = [], s
    for _ in range(5000):
        x = G._step(x)
        seq.append((x * G.MUL) & G.M64)
    assert np.array_equal(G.xorshift_outputs(s, 5000, block=256), np.array(seq, dtype=np.uint64))


def test_lockstep_equals_single_stream():
    seeds = np.array([G.seed_for("sym-uniform", 10), 12345], dtype=np.uint64)
    out = G.xorshift_lockstep(seeds, 50)
    assert np.array_equal(out[0], G.xorshift_outputs(int(seeds[0]), 50))
    assert np.array_equal(out[1], G.xorshift_outputs(12345, 50))


def test_families_deterministic_and_shaped():
    for fam in G.FAMILIES:
        d1, e1 = G.generate(fam, 300)
        d2, e2 = G.generate(fam, 300)
        assert d1.shape == (300,) and e1.shape == (299,)
        assert np.array_equal(d1, d2) and np.array_equal(e1, e2)
    d, e = G.generate("sym-uniform", 1000)
    assert d.min() >= -1 and d.max() < 1 and (e < 0).any() and (e > 0).any()
    d, e = G.generate("wilkinson", 63)
    assert list(d[:21]) == [10, 9, 8, 7, 6, 5, 4, 3, 2, 1, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10]
    assert e[20] == 1e-10 and e[41] == 1e-10 and e[19] == 1.0
    # SPEC.md:567-569
    d, e = G.generate("toeplitz", 3)
    assert list(d) == [2, 2, 2] and list(e) == [0.25, 0.25]
    d, e = G.generate("clustered", 3)
    assert d[1] == 1.0 and e[0] == 1e-4 * (1 + 0.1 * np.cos(0.33))


def test_batch_generator():
    d, e = G.generate_batch("sym-uniform", 3, 16)
    assert d.shape == (3, 16) and e.shape == (3, 15)
    assert not np.array_equal(d[0], d[1])
