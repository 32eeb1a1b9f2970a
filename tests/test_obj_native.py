"""Native OBJ reader (sbr_obj_parse) vs a line-by-line Python restatement of
the reference's reader (E/sceneio.py:129-175) on generated files: number
spellings (exponents, underscores, inf / nan, signs), v/vt/vn corner tokens,
negative indices, comments, tabs, CRLF / CR line ends, injected errors, and
files large enough to be parsed in parallel blocks.  CPU only (host code)."""

import math
import random

import numpy as np
import pytest

from paper_2504_21719_b200 import sceneio
from paper_2504_21719_b200.errors import ParseError


def _py_corner(token, nv, line_no):
    head = token.split("/", 1)[0]
    try:
        raw = int(head)
    except ValueError:
        raise ParseError(f"bad face index {token!r}", line=line_no) from None
    if raw == 0:
        raise ParseError("face indices are 1-based, got 0", line=line_no)
    idx = raw - 1 if raw > 0 else nv + raw
    if not 0 <= idx < nv:
        raise ParseError(f"face index {raw} out of range", line=line_no)
    return idx


def _py_read(path):
    """The checker: the reference's loop, restated (file opened in text mode)."""
    verts, faces = [], []
    with open(path, "r", encoding="ascii") as fh:
        for line_no, line in enumerate(fh, start=1):
            body = line.split("#", 1)[0].strip()
            if not body:
                continue
            parts = body.split()
            if parts[0] == "v":
                if len(parts) < 4:
                    raise ParseError("vertex needs 3 coordinates", line=line_no)
                try:
                    verts.append([float(x) for x in parts[1:4]])
                except ValueError:
                    raise ParseError(f"bad vertex {body!r}", line=line_no) from None
            elif parts[0] == "f":
                if len(parts) < 4:
                    raise ParseError("face needs at least 3 vertices", line=line_no)
                c = [_py_corner(t, len(verts), line_no) for t in parts[1:]]
                for k in range(1, len(c) - 1):
                    faces.append((c[0], c[k], c[k + 1]))
    return (np.asarray(verts, dtype=np.float64).reshape(-1, 3),
            np.asarray(faces, dtype=np.int64).reshape(-1, 3))


def _num(rng):
    r = rng.random()
    x = rng.uniform(-1e3, 1e3)
    if r < 0.3:
        return repr(x)
    if r < 0.4:
        return f"{x:.6e}"
    if r < 0.5:
        return str(rng.randint(-50, 50))
    if r < 0.55:
        return rng.choice(["1_000.5", "2_5e1_0", ".5", "5.", "-0", "+3", "1e-400", "1e400",
                           "1.e5", "-.25E+2", "0001.5"])
    if r < 0.58:
        return rng.choice(["inf", "-Infinity", "nan", "+NaN", "iNf"])
    return f"{x:.17g}"


def _bad_num(rng):
    return rng.choice(["a", "1__0", "_1", "1_", "0x10", "1e", "--1", "1.2.3", "e5", ".", "nan1",
                       "1,5", "infinit"])


def _corner(rng, idx_pos, nv):
    if rng.random() < 0.3:
        tok = str(idx_pos - nv - 1)  # negative (relative) form of the same vertex
    else:
        tok = str(idx_pos)
    r = rng.random()
    if r < 0.2:
        tok += "/1/1"
    elif r < 0.3:
        tok += "//3"
    elif r < 0.35:
        tok += "/7"
    return tok


def _gen(rng, n_lines, p_err=0.0):
    lines, nv = [], 0
    for _ in range(n_lines):
        r = rng.random()
        if p_err and rng.random() < p_err:
            kind = rng.randrange(6)
            if kind == 0:
                lines.append("v 1 2")
            elif kind == 1:
                lines.append(f"v {_num(rng)} {_bad_num(rng)}  {_num(rng)}\t# x")
            elif kind == 2:
                lines.append("f 1 2")
            elif kind == 3 and nv:
                lines.append(f"f 1 {rng.choice(['x', '1x', '/2', '', '1.0'])}/2 1")
            elif kind == 4:
                lines.append("f 0 1 2")
            else:
                lines.append(f"f 1 2 {nv + rng.randint(1, 5)}")
            continue
        if r < 0.45 or nv < 3:
            extra = f" {_num(rng)}" if rng.random() < 0.1 else ""
            sep = rng.choice([" ", "  ", "\t", " \x0b"])
            lines.append(f"v{sep}{_num(rng)}{sep}{_num(rng)} {_num(rng)}{extra}")
            nv += 1
        elif r < 0.75:
            k = rng.choice([3, 3, 3, 4, 5, 8])
            cs = [_corner(rng, rng.randint(1, nv), nv) for _ in range(k)]
            lines.append("f " + " ".join(cs) + (" # tail" if rng.random() < 0.1 else ""))
        elif r < 0.85:
            lines.append(rng.choice(["vn 0 0 1", "vt 0.5 0.5", "g grp", "s off", "usemtl m",
                                     "o obj", "# comment", "", "   ", "vp 1 2 3"]))
        else:
            lines.append("  " + rng.choice(["v", "f"]) + "x 1 2 3")  # unknown keyword
    return lines


def _join(rng, lines):
    out = []
    for ln in lines:
        out.append(ln + rng.choice(["\n", "\n", "\n", "\r\n", "\r"]))
    if rng.random() < 0.5 and out:
        out[-1] = out[-1].rstrip("\r\n")
    return "".join(out)


def _outcome(fn, path):
    try:
        v, t = fn(path)
        return ("ok", v, t)
    except ParseError as e:
        return ("err", str(e), e.line)


def _same(a, b):
    assert a[0] == b[0], (a[:1], b[1:] if b[0] == "err" else None, a[1:] if a[0] == "err" else None)
    if a[0] == "err":
        assert a[1:] == b[1:]
    else:
        np.testing.assert_array_equal(a[1], b[1])  # NaNs compare equal here, -0.0 == 0.0
        assert np.array_equal(np.signbit(a[1]), np.signbit(b[1]))
        np.testing.assert_array_equal(a[2], b[2])


@pytest.mark.parametrize("seed", range(40))
def test_native_obj_matches_python_reader(tmp_path, seed):
    rng = random.Random(seed)
    text = _join(rng, _gen(rng, rng.randint(1, 400), p_err=0.01 if seed % 2 else 0.0))
    p = tmp_path / "m.obj"
    p.write_bytes(text.encode("ascii"))
    _same(_outcome(sceneio._read_obj, p), _outcome(_py_read, p))


@pytest.mark.parametrize("err_at", [None, 0.2, 0.97])
def test_native_obj_parallel_blocks(tmp_path, err_at):
    """Several MB: parsed in parallel blocks; negative indices and range checks
    span block boundaries; the earliest error wins."""
    rng = random.Random(7)
    lines = _gen(rng, 120_000)
    if err_at is not None:
        lines[int(err_at * len(lines))] = "f 1 2 999999999"
        lines[int(0.99 * len(lines))] = "v 1 x 2"
    text = _join(rng, lines)
    assert len(text) > 3 << 20
    p = tmp_path / "big.obj"
    p.write_bytes(text.encode("ascii"))
    _same(_outcome(sceneio._read_obj, p), _outcome(_py_read, p))


def test_native_obj_non_ascii_and_empty(tmp_path):
    p = tmp_path / "e.obj"
    p.write_bytes(b"")
    v, t = sceneio._read_obj(p)
    assert v.shape == (0, 3) and t.shape == (0, 3)
    p.write_bytes("v 0 0 0 # café\n".encode("utf-8"))
    with pytest.raises(UnicodeDecodeError):
        sceneio._read_obj(p)


def test_native_obj_number_spellings(tmp_path):
    p = tmp_path / "n.obj"
    toks = ["1_000.5", "2_5e1_0", ".5", "5.", "-0", "+3", "1e-400", "1e400", "1.e5", "-.25E+2",
            "inf", "-Infinity", "nan", "0.1", "123456789012345678901234567890", "4.9e-324"]
    p.write_text("".join(f"v {a} {a} {a}\n" for a in toks))
    v, _ = sceneio._read_obj(p)
    want = [float(a) for a in toks]
    for row, w in zip(v, want):
        assert (math.isnan(w) and np.isnan(row).all()) or (row == w).all()
        assert bool(np.signbit(row[0])) == (math.copysign(1.0, w) < 0)
