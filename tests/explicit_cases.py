"""Seeded explicit-graph texts (graph.hpp:136-146 format) for the ingestion
tests: well-formed files with random layout (blank lines, comments, tabs,
CR, leading zeros, missing final newline) and single mutations that hit
every ParseError path of parse_explicit_graph (graph.cpp:233-297)."""
from __future__ import annotations

import numpy as np

WS = [b" ", b"  ", b"\t", b" \t ", b"\v", b"\f"]


def _sep(rng) -> bytes:
    return WS[int(rng.integers(0, len(WS)))]


def _id(rng, v: int) -> bytes:
    z = b"0" * int(rng.integers(0, 3)) if rng.random() < 0.1 else b""
    return z + str(v).encode()


def valid_text(rng, n: int, m: int, acc_frac: float = 0.2):
    acc = [int(v) for v in np.flatnonzero(rng.random(n) < acc_frac)]
    if rng.random() < 0.3 and n:
        acc += [int(rng.integers(0, n))]  # duplicates are kept in file order
    edges = rng.integers(0, max(n, 1), size=(m, 2)).tolist() if n else []
    lines = []

    def junk():
        r = rng.random()
        if r < 0.1:
            lines.append(b"")
        elif r < 0.15:
            lines.append(b"# comment " + str(int(rng.integers(0, 99))).encode())
        elif r < 0.18:
            lines.append(_sep(rng) + b"#")

    junk()
    lines.append(_sep(rng) * int(rng.random() < 0.3) + b"graph" + _sep(rng) + str(n).encode()
                 + (b" # vertices" if rng.random() < 0.2 else b""))
    junk()
    lines.append(b"accepting" + b"".join(_sep(rng) + _id(rng, v) for v in acc))
    for s, d in edges:
        junk()
        ln = b"edge" + _sep(rng) + _id(rng, s) + _sep(rng) + _id(rng, d)
        if rng.random() < 0.1:
            ln += _sep(rng) + b"#" + b"x" * int(rng.integers(0, 5))
        if rng.random() < 0.1:
            ln += b"\r"
        lines.append(ln)
    junk()
    text = b"\n".join(lines)
    if rng.random() < 0.7:
        text += b"\n"
    return text, n, acc, edges


def mutated_text(rng, text: bytes, n: int) -> bytes:
    lines = text.split(b"\n")
    nonempty = [i for i, ln in enumerate(lines) if ln.split(b"#")[0].split()]
    kind = int(rng.integers(0, 14))
    pick = lambda k: nonempty[min(k, len(nonempty) - 1)]
    if kind == 0:
        return b""
    if kind == 1:
        return b"\n# only comments\n\n"
    if kind == 2:  # graph line keyword / arity
        lines[pick(0)] = [b"grph 5", b"graph", b"graph 3 4", b"Graph 3"][int(rng.integers(0, 4))]
    elif kind == 3:  # vertex count forms std::stoul accepts or rejects
        lines[pick(0)] = b"graph " + [b"x", b"12abc", b"-1", b"+7", b"99999999999999999999999", b"-"][
            int(rng.integers(0, 6))]
    elif kind == 4:  # no accepting line
        return b"\n".join(lines[: pick(0) + 1]) + b"\n"
    elif kind == 5:
        lines[pick(1)] = b"accept 1"
    elif kind == 6:  # bad accepting ids
        lines[pick(1)] = b"accepting 0 " + [b"1x", b"x1", str(n).encode(), str(n + 1000).encode() + b"z",
                                            b"-1", b"4294967296"][int(rng.integers(0, 6))] + b" 0"
    elif kind == 7 and len(nonempty) > 2:  # edge keyword
        lines[pick(2 + int(rng.integers(0, len(nonempty) - 2)))] = b"edges 0 1"
    elif kind == 8 and len(nonempty) > 2:  # edge arity
        lines[pick(2 + int(rng.integers(0, len(nonempty) - 2)))] = [b"edge 0", b"edge 0 1 2", b"edge"][
            int(rng.integers(0, 3))]
    elif kind == 9 and len(nonempty) > 2:  # bad endpoint ids (non-digit before / after the n break)
        k = pick(2 + int(rng.integers(0, len(nonempty) - 2)))
        lines[k] = b"edge " + [b"0 1y", b"y 0", str(n).encode() + b" 0", b"0 " + str(n * 10 + 7).encode() + b"q",
                               b"0 12#3", b"0x1 0"][int(rng.integers(0, 6))]
    elif kind == 10:  # a second graph line among the edges
        lines.insert(len(lines) - 1, b"graph 3")
    elif kind == 11:  # '#' glued to a token, NUL and high bytes inside tokens
        lines[pick(1)] = b"accepting 0#1 2"
    elif kind == 12 and len(nonempty) > 2:
        lines[pick(2)] = b"edge 0\x00 1"
    else:
        lines.append(b"edge \xff 0")
    return b"\n".join(lines)


def cases(seed: int = 0x0912, count: int = 160):
    rng = np.random.default_rng(seed)
    out = []
    for t in range(count):
        n = int(rng.integers(0, 40)) if t % 7 else int(rng.integers(1, 4))
        m = int(rng.integers(0, 30))
        text, *_ = valid_text(rng, n, m)
        if t % 2 == 1:
            text = mutated_text(rng, text, n)
        out.append(text)
    return out
