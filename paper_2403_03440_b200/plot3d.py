"""ASCII Plot3D (.xyz) single-block grid I/O (reference plot3d.py:22-91).

File layout: an optional block count (a first line holding one token, which
must be 1), the three node counts, then x, y and z, each over all nodes in
Fortran (i fastest) order.  ``#`` starts a comment that runs to the end of
the line.  Errors raise ``ParseError`` carrying the character offset of the
offending token (``byte_offset``; the end of the text when it is truncated);
a block count other than 1 raises ``MultiBlockUnsupported``.

The values are converted in one pass (Python's float(), the reference's
parser) and reshaped with numpy; token offsets are recovered only when a
file is malformed.
"""

from __future__ import annotations

import itertools
import re

import numpy as np

from .errors import MultiBlockUnsupported, ParseError

_TOKEN = re.compile(r"\S+")


def _blank_comments(text):
    """text with every comment replaced by spaces (offsets preserved)."""
    out = []
    for raw in text.splitlines(keepends=True):
        content = raw.splitlines()[0] if raw.splitlines() else ""
        body = content.split("#", 1)[0]
        out.append(body + " " * (len(content) - len(body)) + raw[len(content):])
    return "".join(out)


def _offset(clean, k):
    """Character offset of token k of the comment-free text."""
    m = next(itertools.islice(_TOKEN.finditer(clean), k, None))
    return m.start()


def read_plot3d(path):
    """Nodes (ni, nj, nk, 3) of a single-block ASCII Plot3D file."""
    with open(path, "r", encoding="utf-8") as f:
        text = f.read()
    clean = _blank_comments(text)
    toks = clean.split()
    stripped = text.lstrip()
    head = stripped.splitlines()[0] if stripped.strip() else ""
    pos = 0

    def count(what):
        nonlocal pos
        if pos >= len(toks):
            raise ParseError(f"{what}: file ends early", byte_offset=len(text))
        tok = toks[pos]
        try:
            val = int(tok)
        except ValueError:
            raise ParseError(f"{what}: {tok!r} is not an integer",
                             byte_offset=_offset(clean, pos)) from None
        if val < 1:
            raise ParseError(f"{what}: {val} is not positive", byte_offset=_offset(clean, pos))
        pos += 1
        return val

    if len(head.split()) == 1:
        blocks = count("block count")
        if blocks != 1:
            raise MultiBlockUnsupported(f"{blocks} blocks in file; only single-block grids are read")
    ni, nj, nk = count("ni"), count("nj"), count("nk")
    n = ni * nj * nk
    body = toks[pos:pos + 3 * n]
    try:
        vals = np.fromiter(map(float, body), dtype=float, count=len(body))
    except ValueError:
        for k, tok in enumerate(body):
            try:
                float(tok)
            except ValueError:
                raise ParseError(f"coordinate {tok!r} is not a number",
                                 byte_offset=_offset(clean, pos + k)) from None
        raise
    if len(body) < 3 * n:
        raise ParseError(f"file ends after {len(body)} of {3 * n} coordinates",
                         byte_offset=len(text))
    if len(toks) > pos + 3 * n:
        raise ParseError("data after the single block", byte_offset=_offset(clean, pos + 3 * n))
    return np.stack([vals[c * n:(c + 1) * n].reshape((ni, nj, nk), order="F") for c in range(3)],
                    axis=-1)


def write_plot3d(path, nodes):
    """Write nodes (ni, nj, nk, 3) as a one-block ASCII Plot3D file, five
    values per line at full double precision (%.17e round-trips exactly)."""
    a = np.asarray(nodes, dtype=float)
    ni, nj, nk = a.shape[:3]
    lines = ["1", f"{ni} {nj} {nk}"]
    for c in range(3):
        flat = a[..., c].ravel(order="F")
        lines.extend(" ".join("%.17e" % v for v in flat[s:s + 5]) for s in range(0, flat.size, 5))
    with open(path, "w", encoding="utf-8") as f:
        f.write("\n".join(lines) + "\n")


__all__ = ["read_plot3d", "write_plot3d"]
