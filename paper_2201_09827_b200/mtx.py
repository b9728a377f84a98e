"""Matrix Market ingestion for the sweep layer (reference matgen.py:29-38,
113-236): real/integer ``coordinate`` or ``array`` files, ``general`` or
``symmetric``, read into a dense float64 matrix (the solver's input layout).

Behaviour follows the reference reader: symmetric storage is mirrored,
duplicate coordinate entries are summed, array data is column-major, and
malformed input raises ``ParseError`` carrying the 1-based line number;
complex / pattern / skew / hermitian files raise ``UnsupportedField``.
"""

from __future__ import annotations

import numpy as np

__all__ = ["ParseError", "UnsupportedField", "read_matrix_market", "write_matrix_market"]


class ParseError(Exception):
    """Malformed Matrix Market input; ``line_no`` is the offending line."""

    def __init__(self, line_no: int, message: str):
        self.line_no = line_no
        super().__init__(f"line {line_no}: {message}")


class UnsupportedField(Exception):
    """A field or symmetry this reader does not accept."""


def _int(tok: str, line_no: int) -> int:
    try:
        return int(tok)
    except ValueError:
        raise ParseError(line_no, f"expected integer, got {tok!r}") from None


def _data_lines(lines: list, start: int):
    """(1-based line number, stripped text) of every data line from ``start``."""
    for idx in range(start, len(lines)):
        text = lines[idx].strip()
        if text and not text.startswith("%"):
            yield idx + 1, text


def _header(lines: list) -> tuple:
    if not lines:
        raise ParseError(1, "empty file")
    head = lines[0].split()
    if len(head) < 5 or head[0] not in ("%%MatrixMarket", "%MatrixMarket"):
        raise ParseError(1, "missing %%MatrixMarket header")
    obj, layout, field, symmetry = (t.lower() for t in head[1:5])
    if obj != "matrix":
        raise ParseError(1, f"unsupported object {obj!r}")
    if layout not in ("coordinate", "array"):
        raise ParseError(1, f"unsupported layout {layout!r}")
    if field not in ("real", "integer"):
        raise UnsupportedField(f"field {field!r} is not supported")
    if symmetry not in ("general", "symmetric"):
        raise UnsupportedField(f"symmetry {symmetry!r} is not supported")
    return layout, symmetry == "symmetric"


def read_matrix_market(path) -> np.ndarray:
    with open(path, "r", encoding="ascii") as fh:
        lines = fh.readlines()
    layout, symmetric = _header(lines)
    body = _data_lines(lines, 1)
    try:
        size_no, size_text = next(body)
    except StopIteration:
        raise ParseError(len(lines), "missing size line") from None
    size = size_text.split()

    if layout == "coordinate":
        if len(size) != 3:
            raise ParseError(size_no, "coordinate size line needs rows cols nnz")
        rows, cols, nnz = (_int(t, size_no) for t in size)
        a = np.zeros((rows, cols))
        count = 0
        for no, text in body:
            toks = text.split()
            if len(toks) != 3:
                raise ParseError(no, "expected 'row col value'")
            r, c = _int(toks[0], no), _int(toks[1], no)
            try:
                v = float(toks[2])
            except ValueError:
                raise ParseError(no, f"bad value {toks[2]!r}") from None
            if not (1 <= r <= rows and 1 <= c <= cols):
                raise ParseError(no, f"index ({r},{c}) out of range")
            a[r - 1, c - 1] += v
            if symmetric and r != c:
                a[c - 1, r - 1] += v
            count += 1
        if count != nnz:
            raise ParseError(len(lines), f"expected {nnz} entries, found {count}")
        return a

    if len(size) != 2:
        raise ParseError(size_no, "array size line needs rows cols")
    rows, cols = (_int(t, size_no) for t in size)
    vals = []
    for no, text in body:
        try:
            vals.append(float(text.split()[0]))
        except ValueError:
            raise ParseError(no, f"bad value {text!r}") from None
    if symmetric:
        want = rows * (rows + 1) // 2
        if rows != cols or len(vals) != want:
            raise ParseError(len(lines), f"expected {want} entries for symmetric array")
        a = np.zeros((rows, cols))
        lower = np.tril_indices(rows)
        # column-major lower triangle: order by column, then row
        order = np.lexsort((lower[0], lower[1]))
        r_idx, c_idx = lower[0][order], lower[1][order]
        a[r_idx, c_idx] = vals
        a[c_idx, r_idx] = vals
        return a
    if len(vals) != rows * cols:
        raise ParseError(len(lines), f"expected {rows * cols} entries, found {len(vals)}")
    return np.asarray(vals, dtype=np.float64).reshape(cols, rows).T.copy()


def write_matrix_market(path, a, comment: str | None = None) -> None:
    """Dense matrix to coordinate/general (zeros dropped), values round-trip exactly."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError("write_matrix_market requires a 2-D matrix")
    rr, cc = np.nonzero(a)
    out = ["%%MatrixMarket matrix coordinate real general"]
    if comment:
        out += [f"% {line}" for line in comment.splitlines()]
    out.append(f"{a.shape[0]} {a.shape[1]} {len(rr)}")
    out += [f"{r + 1} {c + 1} {float(a[r, c])!r}" for r, c in zip(rr, cc)]
    with open(path, "w", encoding="ascii") as fh:
        fh.write("\n".join(out) + "\n")
