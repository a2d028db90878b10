"""The parallel G-set parser (csrc/host/graph.cpp) on inputs
large enough to be cut into one piece per host thread (> 1 MB): the result and
the reported error (class, message and line number: the first offending line
in file order, reference graph.cpp:81-128) match a serial restatement of the
reference parser, including duplicates whose first occurrence lies in an
earlier piece and errors in later pieces. CPU only."""
import re

import numpy as np
import pytest

import paper_1908_00210_b200 as pi


def serial_reference(text):
    """graph.cpp:81-128 restated: (n, edges) or (message, line)."""
    lines = text.split("\n")
    if text.endswith("\n"):
        lines = lines[:-1]
    no = 0
    it = iter(lines)
    head = None
    for ln in it:
        no += 1
        s = ln.strip(" \t\r")
        if not s or s[0] in "%#":
            continue
        head = s.split()
        break
    n, m = int(head[0]), int(head[1])
    seen, edges = set(), []
    for ln in it:
        no += 1
        s = ln.strip(" \t\r")
        if not s or s[0] in "%#":
            continue
        t = s.split()
        if len(t) != 3 or not all(re.fullmatch(r"-?\d+", x) for x in t):
            return ("edge line must be", no)
        u, v, w = (int(x) for x in t)
        if not (1 <= u <= n and 1 <= v <= n):
            return ("endpoint out of range", no)
        if u == v:
            return ("self-loop", no)
        if not (-2 ** 31 <= w < 2 ** 31):
            return ("weight out of range", no)
        k = (min(u, v), max(u, v))
        if k in seen:
            return ("duplicate edge", no)
        seen.add(k)
        edges.append((u - 1, v - 1, w))
    if len(edges) != m:
        return ("header announces", None)
    return n, edges


@pytest.fixture(scope="module")
def big_text():
    g = pi.random_graph(60000, 240000, 99)  # ~3.5 MB of text
    return g.to_gset()


def lines_of(text):
    return text.split("\n")


def check(text):
    ref = serial_reference(text)
    if isinstance(ref[0], str):
        msg, line = ref
        with pytest.raises(pi.ParseError) as ei:
            pi.Graph.parse_gset(text)
        assert msg in str(ei.value), (str(ei.value), msg)
        if line is not None:
            assert f"line {line}" in str(ei.value), (str(ei.value), line)
    else:
        g = pi.Graph.parse_gset(text)
        n, edges = ref
        assert g.num_nodes == n and g.num_edges == len(edges)
        h = pi.Graph.from_edges(n, edges)
        for v in range(0, n, max(1, n // 997)):  # identical rows, insertion order
            assert g.neighbors(v) == h.neighbors(v)


def test_parallel_parse_matches_serial(big_text):
    check(big_text)
    assert len(big_text) > (1 << 20)


@pytest.mark.parametrize("where", [0.1, 0.5, 0.93])
def test_duplicate_across_pieces(big_text, where):
    ls = lines_of(big_text)
    i = int(where * (len(ls) - 2)) + 1
    ls.insert(len(ls) - 1, ls[i])  # repeat an early edge at the end (header count now off by one too)
    check("\n".join(ls))


def test_first_error_in_file_order(big_text):
    ls = lines_of(big_text)
    n1 = len(ls)
    ls[int(0.8 * n1)] = "1 2"  # a malformed line late ...
    ls[int(0.6 * n1)] = ls[int(0.05 * n1)]  # ... after a duplicate whose first occurrence is early
    check("\n".join(ls))
    ls2 = lines_of(big_text)
    ls2[int(0.3 * n1)] = "7 7 1"  # self-loop before the duplicate
    ls2[int(0.6 * n1)] = ls2[int(0.05 * n1)]
    check("\n".join(ls2))


@pytest.mark.parametrize("bad", ["1 60001 1", "3 4 99999999999", "x 1 2", "5 5 5"])
def test_errors_in_late_pieces(big_text, bad):
    ls = lines_of(big_text)
    ls[int(0.97 * len(ls))] = bad
    check("\n".join(ls))


def test_comments_blank_lines_and_crlf_across_cuts(big_text):
    ls = lines_of(big_text)
    out = []
    for k, ln in enumerate(ls):
        out.append(ln + ("\r" if k % 7 == 3 and ln else ""))
        if k % 1000 == 999:
            out.append("% comment")
            out.append("")
    check("\n".join(out))
