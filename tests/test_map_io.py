"""LEGOMAP1 map files through the C ABI (lgs_map_file_*) against an
independent struct-based restatement of proj/src/gaussian_map.cpp:196-259 and the reference's own
map-file tests (proj/tests/test_map.cpp:118-170): empty round trip, bitwise round trip,
dimension mismatch / truncation / bad magic as distinct IoErrors.  Host-only: no GPU needed."""
import os
import struct

import numpy as np
import pytest

from paper_2511_16144_b200 import _lib
from paper_2511_16144_b200 import renderer as R

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "map_small.legomap")


def py_write(path, scene, anchors):
    """gaussian_map.cpp:196-218, restated with struct."""
    d, n = scene["feat"].shape
    with open(path, "wb") as f:
        f.write(b"LEGOMAP1")
        f.write(struct.pack("<IQ", d, n))
        for i in range(n):
            x, y, z, w = (float(v) for v in scene["rot"][i])
            f.write(struct.pack("<3f", *scene["pos"][i]))
            f.write(struct.pack("<4f", w, x, y, z))
            f.write(struct.pack("<3f", *scene["log_s"][i]))
            f.write(struct.pack("<f", scene["opac"][i]))
            f.write(struct.pack("<3f", *scene["sh"][i, 0]))
            f.write(struct.pack(f"<{d}f", *scene["feat"][:, i]))
            f.write(struct.pack("<Q", int(anchors[i])))


def random_scene(n, d, seed):
    r = np.random.default_rng(seed)
    q = r.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return {"pos": r.normal(size=(n, 3)).astype(np.float32), "rot": q.astype(np.float32),
            "log_s": r.normal(-3, 0.5, (n, 3)).astype(np.float32), "opac": r.normal(size=n).astype(np.float32),
            "sh": r.uniform(0, 1, (n, 1, 3)).astype(np.float32), "feat": r.normal(size=(d, n)).astype(np.float32)}


def test_empty_map_round_trip(tmp_path):
    p = str(tmp_path / "empty.bin")
    R.map_file_write(p, random_scene(0, 16, 0))
    assert R.map_file_info(p) == (16, 0)
    scene, anchors = R.map_file_read(p)
    assert scene["feat"].shape == (16, 0) and anchors.size == 0


def test_round_trip_is_bitwise_and_matches_struct_restatement(tmp_path):
    scene = random_scene(1000, 16, 6)
    scene["rot"] = (scene["rot"] / np.linalg.norm(scene["rot"].astype(np.float64), axis=1, keepdims=True)).astype(
        np.float32)
    anchors = (np.arange(1000) % 7).astype(np.uint64)
    a, b = str(tmp_path / "lib.bin"), str(tmp_path / "py.bin")
    R.map_file_write(a, scene, anchors)
    py_write(b, scene, anchors)
    assert open(a, "rb").read() == open(b, "rb").read()
    back, back_anchors = R.map_file_read(a)
    assert np.array_equal(back_anchors, anchors)
    for k in scene:
        unit = np.abs(np.linalg.norm(scene["rot"].astype(np.float64), axis=1) - 1.0) <= 1e-6
        if k == "rot":
            assert np.array_equal(back[k][unit], scene[k][unit])
        else:
            assert np.array_equal(back[k], scene[k]), k


def test_off_unit_rotation_is_renormalized(tmp_path):
    scene = random_scene(3, 4, 1)
    scene["rot"][1] *= 3.0
    p = str(tmp_path / "q.bin")
    py_write(p, scene, np.zeros(3, np.uint64))
    back, _ = R.map_file_read(p)
    assert np.linalg.norm(back["rot"][1].astype(np.float64)) == pytest.approx(1.0, abs=1e-6)


def test_golden_fixture():
    """tests/golden/map_small.legomap (3 Gaussians, d = 4, written by tests/golden/make_golden.py
    with the struct restatement above)."""
    scene, anchors = R.map_file_read(GOLDEN)
    assert scene["pos"].shape == (3, 3) and list(anchors) == [0, 5, 7]
    assert np.array_equal(scene["pos"][1], np.array([1.5, -2.0, 3.25], np.float32))
    assert np.array_equal(scene["rot"][0], np.array([0.0, 0.0, 0.0, 1.0], np.float32))  # identity, x,y,z,w
    assert np.array_equal(scene["feat"][:, 2], np.array([0.5, -0.5, 0.25, 1.0], np.float32))


def test_errors_match_reference(tmp_path):
    """test_map.cpp:148-170: dimension mismatch, truncation and bad magic raise distinct IoErrors."""
    p = str(tmp_path / "dim.bin")
    R.map_file_write(p, random_scene(1, 32, 7))
    with pytest.raises(_lib.LgsIoError, match="dimension mismatch"):
        R.map_file_read(p, expected_dim=16)
    os.truncate(p, os.path.getsize(p) - 8)
    with pytest.raises(_lib.LgsIoError, match="truncated"):
        R.map_file_read(p)
    with open(p, "wb") as f:
        f.write(b"NOTAMAP!" + b"\0" * 64)
    with pytest.raises(_lib.LgsIoError, match="magic"):
        R.map_file_read(p)
    with pytest.raises(OSError, match="cannot open"):
        R.map_file_read(str(tmp_path / "missing.bin"))
    sh3 = dict(random_scene(2, 4, 1), sh=np.zeros((2, 16, 3), np.float32))
    with pytest.raises(ValueError):
        R.map_file_write(str(tmp_path / "sh3.bin"), sh3)


def test_huge_declared_count_is_a_truncation_error(tmp_path):
    """A corrupt header declaring 2^60 Gaussians: the file is sized against the count before any
    buffer is sized from it (the reference reads record by record and raises "map file truncated";
    sizing vectors first would throw std::bad_alloc through the C ABI)."""
    import struct
    p = str(tmp_path / "huge.bin")
    R.map_file_write(p, random_scene(3, 4, 5))
    with open(p, "r+b") as f:
        f.seek(12)
        f.write(struct.pack("<Q", 1 << 60))
    with pytest.raises(_lib.LgsIoError, match="truncated reading"):
        R.map_file_info(p)
    with pytest.raises(_lib.LgsIoError, match="truncated reading"):
        R.map_file_read(p)
    # a count one past the records: the error names the field the reader runs out in
    with open(p, "r+b") as f:
        f.seek(12)
        f.write(struct.pack("<Q", 4))
    with pytest.raises(_lib.LgsIoError, match="truncated reading position"):
        R.map_file_read(p)
