"""Point-set and image files against the reference's own
save/load functions (imaging.cpp:235-304, 433-494) compiled in oracle/_ref:
files written by either side read back identically on the other, and the
reference's error codes come back for broken files.  CPU only."""
import os

import numpy as np
import pytest


@pytest.fixture
def gmi():
    import paper_2012_13257_b200 as g

    return g


def _points(seed, n, ch):
    rng = np.random.default_rng(seed)
    pos = rng.uniform(-3, 50, (n, 2)).astype(np.float32).astype(np.float64)
    col = rng.uniform(0, 1, (n, ch)).astype(np.float32).astype(np.float64)
    return pos, col


@pytest.mark.parametrize("ch", [1, 3])
def test_point_set_round_trip_with_reference(gmi, ref, tmp_path, ch):
    pos, col = _points(ch, 257, ch)
    ours = str(tmp_path / "ours.csv")
    theirs = str(tmp_path / "theirs.csv")
    gmi.save_point_set(gmi.PointSet(pos, col), ours)
    ref.save_point_set(pos, col, theirs)
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    rp, rc = ref.load_point_set(ours)
    ps = gmi.load_point_set(theirs)
    assert np.array_equal(rp, pos) and np.array_equal(rc, col)
    assert np.array_equal(ps.positions, pos) and np.array_equal(ps.colors, col)


@pytest.mark.parametrize("text,code", [
    ("x,y,q\n1,2,0.5\n", 12),              # header
    ("x,y,v\n1,2\n", 12),                  # field count
    ("x,y,v\n1, 2,0.5\n3 ,4,0.5\n", 12),    # space before a comma
    ("x,y,v\n1,2,abc\n", 12),              # bad number
    ("x,y,v\n1,2,1.5\n", 2),               # colour out of [0,1]
    ("x,y,v\n\n", 3),                      # empty
    ("x,y,r,g,b\r\n1,2,0.1,0.2,0.3 \r\n\r\n0x1p-2,5e-1,1,0,inf\n", 1),  # non-finite colour
])
def test_point_set_errors_match_reference(gmi, ref, tmp_path, text, code):
    import oracle

    path = str(tmp_path / "p.csv")
    with open(path, "w", newline="") as f:
        f.write(text)
    with pytest.raises(oracle.OracleError) as r:
        ref.load_point_set(path)
    with pytest.raises(gmi.GmiError) as g:
        gmi.load_point_set(path)
    assert r.value.code == code == g.value.code


def test_point_set_parsing_matches_reference(gmi, ref, tmp_path):
    path = str(tmp_path / "p.csv")
    with open(path, "w", newline="") as f:
        f.write("x,y,r,g,b\r\n1, 2.5e0,0.1,0.2,0.3  \r\n\n-0x1p-2,+.5,1,0,1e-300\n")
    rp, rc = ref.load_point_set(path)
    ps = gmi.load_point_set(path)
    assert np.array_equal(ps.positions, rp.astype(np.float32))
    assert np.array_equal(ps.colors, rc.astype(np.float32))
    with pytest.raises(gmi.GmiError) as e:
        gmi.load_point_set(str(tmp_path / "missing.csv"))
    assert e.value.code == 14


@pytest.mark.parametrize("ext,ch", [(".ppm", 3), (".pnm", 1), (".pgm", 1), (".PPM", 3)])
def test_image_files_match_reference(gmi, ref, tmp_path, ext, ch):
    rng = np.random.default_rng(3)
    img = rng.uniform(-0.1, 1.1, (13, 17, ch))
    img[0, 0, 0] = 0.5 / 255.0 * 3  # a rounding tie (lround: half away from zero)
    ours = str(tmp_path / ("ours" + ext))
    theirs = str(tmp_path / ("theirs" + ext))
    gmi.save_image(img, ours)
    ref.save_image(img, theirs)
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    assert np.array_equal(gmi.load_image(theirs), ref.load_image(theirs))


def test_image_header_comments_maxval_and_errors(gmi, ref, tmp_path):
    import oracle

    path = str(tmp_path / "c.pgm")
    data = bytes(range(12))
    with open(path, "wb") as f:
        f.write(b"P5\n# a comment\n4 # width\n3\n100\n" + data)
    assert np.array_equal(gmi.load_image(path), ref.load_image(path))
    cases = {
        "trunc.pgm": (b"P5\n4 3\n255\n" + data[:5], 12),
        "max.pgm": (b"P5\n4 3\n1000\n" + data, 11),
        "bad.pgm": (b"P5\n4 x\n255\n" + data, 12),
        "x.png": (b"\x89PNG\r\n\x1a\n" + data, 11),
        "x.bin": (b"GIF89a" + data, 11),
    }
    for name, (blob, code) in cases.items():
        p = str(tmp_path / name)
        with open(p, "wb") as f:
            f.write(blob)
        with pytest.raises(oracle.OracleError) as r:
            ref.load_image(p)
        with pytest.raises(gmi.GmiError) as g:
            gmi.load_image(p)
        assert r.value.code == code == g.value.code, name
    for name, img, code in [("a.png", np.zeros((2, 2, 1)), 11), ("a.pgm", np.zeros((2, 2, 3)), 11),
                            ("a.tif", np.zeros((2, 2, 1)), 11), ("a.ppm", np.zeros((2, 2, 2)), 8)]:
        with pytest.raises(oracle.OracleError) as r:
            ref.save_image(img, str(tmp_path / name))
        with pytest.raises(gmi.GmiError) as g:
            gmi.save_image(img, str(tmp_path / name))
        assert r.value.code == code == g.value.code, name
