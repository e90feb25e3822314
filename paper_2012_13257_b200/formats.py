"""Point-set and image files, host side, numpy only.

Mirrors the reference's imaging.cpp formats so files written by either side
read back on the other:

* point sets: CSV with header ``x,y,r,g,b`` (3 channels) or ``x,y,v`` (1
  channel), values printed with ``%.17g`` (save_point_set / load_point_set,
  imaging.cpp:433-494, format_double imaging.cpp:16-20, parse_csv_row
  imaging.cpp:392-420);
* images: binary PNM — P6 for ``.ppm``/``.pnm`` (grey replicated to RGB),
  P5 for ``.pgm`` (1 channel only), maxval <= 255, ``#`` comments in the
  header, values ``byte / maxval`` in, ``clamp(lround(v * 255), 0, 255)`` out
  (load_pnm / save_pnm imaging.cpp:32-124, load_image / save_image
  imaging.cpp:235-304).  PNG needs libpng, optional in the reference
  (GMI_HAVE_PNG): here it is UnsupportedFormat, as in a reference build
  without it.

Errors are GmiError with the reference's codes (1 + gmi::ErrorCode):
IoError, CorruptFile, UnsupportedFormat, InvalidDimensions, and the point-set
validation of require_valid (core.cpp:55-102; the file format holds 1 or 3
channels).  Positions and colours of a loaded PointSet are held in fp32 like
every PointSet of this package (exact for fp32-representable values).
"""
from __future__ import annotations

import re

import numpy as np

E_SHAPE, E_INVALID_DIM, E_UNSUPPORTED, E_CORRUPT, E_IO = 4, 8, 11, 12, 14


def _err(code, msg):
    from . import GmiError

    return GmiError(code, msg)


# strtod's accepted forms after leading whitespace: decimal, hex, inf, nan
_NUM = re.compile(r"[ \t\n\v\f\r]*([+-]?(?:0[xX](?:[0-9a-fA-F]+\.?[0-9a-fA-F]*|\.[0-9a-fA-F]+)"
                  r"(?:[pP][+-]?\d+)?|(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?|inf(?:inity)?|nan))",
                  re.IGNORECASE)


def _parse_row(line: str, line_no: int, path: str):
    """parse_csv_row (imaging.cpp:392-420): strtod per field, ',' between
    fields, only spaces / CR after the last one; else CorruptFile."""
    vals, p, n = [], 0, len(line)
    while True:
        m = _NUM.match(line, p)
        if not m:
            raise _err(E_CORRUPT, f"{path}: bad number at line {line_no}")
        tok = m.group(1)
        vals.append(float.fromhex(tok) if "x" in tok.lower() else float(tok))
        p = m.end()
        if p < n and line[p] == ",":
            p += 1
            continue
        while p < n and line[p] in " \r":
            p += 1
        if p == n:
            return vals
        raise _err(E_CORRUPT, f"{path}: trailing garbage at line {line_no}")


def save_point_set(points, path: str) -> None:
    """save_point_set (imaging.cpp:433-452)."""
    from . import PointSet

    if not isinstance(points, PointSet):
        raise TypeError("points must be a PointSet")
    ch = points.channels
    if ch not in (1, 3):  # require_valid (core.cpp:60-64)
        raise _err(E_SHAPE, f"channels must be 1 or 3, got {ch}")
    pos, col = points.positions, points.colors
    try:
        with open(path, "w", newline="\n") as f:
            f.write("x,y,r,g,b\n" if ch == 3 else "x,y,v\n")
            for i in range(len(points)):
                f.write(",".join("%.17g" % v for v in (pos[i, 0], pos[i, 1], *col[i])) + "\n")
    except OSError:
        raise _err(E_IO, f"cannot open for writing: {path}") from None


def load_point_set(path: str):
    """load_point_set (imaging.cpp:454-494) -> PointSet."""
    from . import PointSet

    try:
        with open(path, "rb") as f:
            data = f.read().decode("latin-1")
    except OSError:
        raise _err(E_IO, f"cannot open file: {path}") from None
    lines = data.split("\n")
    header = lines[0].rstrip("\r\n")
    if header == "x,y,r,g,b":
        ch = 3
    elif header == "x,y,v":
        ch = 1
    else:
        raise _err(E_CORRUPT, f'{path}: expected header "x,y,r,g,b" or "x,y,v"')
    rows = []
    for k, line in enumerate(lines[1:], start=2):
        line = line.rstrip("\r")
        if not line:
            continue
        v = _parse_row(line, k, path)
        if len(v) != 2 + ch:
            raise _err(E_CORRUPT, f"{path}: expected {2 + ch} fields at line {k}")
        rows.append(v)
    arr = np.array(rows, np.float64).reshape(-1, 2 + ch)
    return PointSet(arr[:, :2], arr[:, 2:])


def _pnm_token(buf: bytes, i: int, path: str):
    """pnm_token (imaging.cpp:32-56): skip whitespace and '#' comment lines,
    read a decimal; the byte after the digits is consumed."""
    n = len(buf)
    while True:
        while i < n and chr(buf[i]).isspace():
            i += 1
        if i < n and buf[i] == ord("#"):
            while i < n and buf[i] != ord("\n"):
                i += 1
            continue
        break
    if i >= n or not chr(buf[i]).isdigit():
        raise _err(E_CORRUPT, f"malformed PNM header in {path}")
    v = 0
    while i < n and chr(buf[i]).isdigit():
        v = v * 10 + buf[i] - ord("0")
        i += 1
    return v, i + 1


def load_image(path: str) -> np.ndarray:
    """load_image (imaging.cpp:235-270) -> H x W x C float64 in [0, 1]."""
    try:
        with open(path, "rb") as f:
            buf = f.read()
    except OSError:
        raise _err(E_IO, f"cannot open file: {path}") from None
    if len(buf) >= 2 and buf[0] == ord("P") and buf[1] in (ord("5"), ord("6")):
        ch = 3 if buf[1] == ord("6") else 1
        w, i = _pnm_token(buf, 2, path)
        h, i = _pnm_token(buf, i - 1, path)
        maxval, i = _pnm_token(buf, i - 1, path)
        if w < 1 or h < 1:
            raise _err(E_CORRUPT, f"bad PNM dimensions in {path}")
        if maxval < 1 or maxval > 255:
            raise _err(E_UNSUPPORTED, f"PNM maxval {maxval} unsupported (need <= 255): {path}")
        n = w * h * ch
        raw = np.frombuffer(buf, np.uint8, count=min(n, max(0, len(buf) - i)), offset=min(i, len(buf)))
        if raw.size != n:
            raise _err(E_CORRUPT, f"truncated PNM data in {path}")
        return (raw.astype(np.float64) * (1.0 / maxval)).reshape(h, w, ch)
    if len(buf) >= 8 and buf[:8] == b"\x89PNG\r\n\x1a\n":
        raise _err(E_UNSUPPORTED, f"PNG support not compiled in: {path}")
    raise _err(E_UNSUPPORTED, f"unrecognized image format: {path}")


def save_image(image, path: str) -> None:
    """save_image (imaging.cpp:272-304) for .ppm / .pnm / .pgm."""
    img = np.asarray(image, np.float64)
    if img.ndim == 2:
        img = img[:, :, None]
    if img.ndim != 3 or img.shape[0] < 1 or img.shape[1] < 1 or img.shape[2] not in (1, 3):
        raise _err(E_INVALID_DIM, "image must be nonempty with 1 or 3 channels")
    low = path.lower()
    if low.endswith(".ppm") or low.endswith(".pnm"):
        out_ch = 3
    elif low.endswith(".pgm"):
        if img.shape[2] != 1:
            raise _err(E_UNSUPPORTED, f"cannot write RGB data as PGM: {path}")
        out_ch = 1
    elif low.endswith(".png"):
        raise _err(E_UNSUPPORTED, f"PNG support not compiled in: {path}")
    else:
        raise _err(E_UNSUPPORTED, f"unsupported image extension: {path}")
    h, w, ch = img.shape
    src = np.minimum(np.arange(out_ch), ch - 1)  # grey replicated to RGB
    v = img[:, :, src] * 255.0
    # std::lround: half away from zero; NaN -> LONG_MIN -> clamped to 0
    q = np.where(np.isnan(v), -1.0, np.sign(v) * np.floor(np.abs(v) + 0.5))
    raw = np.clip(q, 0, 255).astype(np.uint8)
    try:
        with open(path, "wb") as f:
            f.write(("P6" if out_ch == 3 else "P5").encode() + b"\n" +
                    f"{w} {h}\n255\n".encode() + raw.tobytes())
    except OSError:
        raise _err(E_IO, f"cannot open for writing: {path}") from None
