"""scenes.RefRng (the reference's lego::Rng as a vectorized numpy generator, random.hpp:12-50)
against the oracle's C restatement (oracle/lgs_oracle.c orc_rng_*, pinned to the C++ standard's
mt19937_64 value in tests/test_oracle_ext.py): the u64 stream, uniform(), uniform(lo, hi),
uniform_int and the Box-Muller normal() with its cached second value, across calls of odd sizes."""
import numpy as np

from paper_2511_16144_b200 import scenes


def test_u64_stream_and_standard_value(oracle):
    r = scenes.RefRng(5489)
    assert int(r.next_u64(10000)[-1]) == 9981545732273789042  # [rand.predef]
    a, b = scenes.RefRng(1001), oracle.Rng(1001)
    got = np.concatenate([a.next_u64(k) for k in (1, 311, 312, 700, 5)])
    want = np.array([b.next_u64() for _ in range(got.size)], dtype=np.uint64)
    assert np.array_equal(got, want)


def test_transforms_match_the_reference_rng(oracle):
    a, b = scenes.RefRng(77), oracle.Rng(77)
    for k in (3, 1, 8, 5):  # odd sizes: the normal() spare carries across calls
        assert np.array_equal(a.uniform(-2.0, 3.0, k), np.array([b.uniform(-2.0, 3.0) for _ in range(k)]))
        assert np.array_equal(a.standard_normal(k), np.array([b.normal() for _ in range(k)]))
    ints = a.integers(0, 200, 9)
    want = np.array([int(b.uniform() * 200) for _ in range(9)])
    assert np.array_equal(ints, want)


def test_reference_rng_scene_has_the_config_shapes():
    s, cams, info = scenes.make_config("c0", rng="reference")
    p, _, _ = scenes.make_config("c0")
    assert info["rng"] == "reference" and {k: v.shape for k, v in s.items()} == {k: v.shape for k, v in p.items()}
    assert not np.array_equal(s["pos"], p["pos"])
    s2, _, _ = scenes.make_config("c0", rng="reference")
    assert all(np.array_equal(s[k], s2[k]) for k in s)  # reproducible
