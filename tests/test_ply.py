"""PLY loader parity with the reference (§8f row 4): every fixture in
tests/golden/ply.npz was loaded by the reference's own load_ply
(tests/golden/make_ply_golden.py); the B200 package must return the same
arrays bit for bit, or raise PlyParseError with the same message and byte
offset.  Plus save/load round trips (pkg/tests/test_acceptance.py:261-272)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN

from paper_2502_11618_b200.errors import PlyParseError
from paper_2502_11618_b200.io.ply import load_ply, save_ply

_G = np.load(os.path.join(GOLDEN, "ply.npz"))
CASES = sorted({k.split("__")[0] for k in _G.files})


@pytest.mark.parametrize("name", CASES)
def test_load_matches_reference(name, tmp_path):
    p = tmp_path / f"{name}.ply"
    p.write_bytes(_G[f"{name}__bytes"].tobytes())
    if f"{name}__pos" in _G.files:
        c = load_ply(p)
        assert np.array_equal(c.positions, _G[f"{name}__pos"])
        assert np.array_equal(c.colors, _G[f"{name}__col"])
    else:
        assert f"{name}__err" in _G.files, name
        with pytest.raises(PlyParseError) as ei:
            load_ply(p)
        assert str(ei.value) == str(_G[f"{name}__err"])
        assert ei.value.offset == int(_G[f"{name}__off"])


def test_save_matches_reference_bytes(tmp_path):
    from paper_2502_11618_b200 import PointCloud

    c = PointCloud(_G["saved_bin__pos"], _G["saved_bin__col"])
    for binary, key in ((True, "saved_bin__bytes"), (False, "saved_ascii__bytes")):
        p = tmp_path / "out.ply"
        save_ply(c, p, binary=binary)
        assert p.read_bytes() == _G[key].tobytes()


def test_roundtrip_both_formats(rng, tmp_path):
    from paper_2502_11618_b200 import PointCloud

    c = PointCloud((rng.random((777, 3)) * 40 - 20).astype(np.float32),
                   rng.integers(0, 256, (777, 3), dtype=np.uint8))
    save_ply(c, tmp_path / "a.ply", binary=False)
    save_ply(c, tmp_path / "b.ply", binary=True)
    a, b = load_ply(tmp_path / "a.ply"), load_ply(tmp_path / "b.ply")
    for x in (a, b):
        assert np.array_equal(x.positions, c.positions) and np.array_equal(x.colors, c.colors)
