"""NEXT-4 host runtime (§3.4):
the Kahn task scheduler of the step and the bounded asynchronous writer of the
compute / postprocess split.  Host-only entry points of libdpd.so -- no GPU needed.

Pins (not the implementation re-typed): the order is checked against the DEFINITION of a
topological order (every edge respected, every task once) and, on small random DAGs,
against a brute-force enumeration of all permutations (Kahn with an earliest-added tie
break must return the lexicographically smallest topological order); cycles of every length
are rejected; the writer is checked by its observable contract (files, counts, timing)."""
import itertools
import os
import time

import numpy as np
import pytest

from paper_1911_04712_b200 import capi


def random_dag(rng, n, p):
    perm = rng.permutation(n)  # hidden topological order
    edges = [(int(perm[i]), int(perm[j])) for i in range(n) for j in range(i + 1, n) if rng.random() < p]
    return edges


def kahn(n, edges):
    g = capi.TaskGraph()
    ids = [g.add(f"t{k}", k % 3) for k in range(n)]
    assert ids == list(range(n))
    for a, b in edges:
        g.edge(a, b)
    return g.order()


def test_order_is_a_topological_order():
    rng = np.random.default_rng(7)
    for _ in range(50):
        n = int(rng.integers(1, 40))
        edges = random_dag(rng, n, 0.15)
        order = kahn(n, edges)
        assert sorted(order) == list(range(n))
        pos = {t: k for k, t in enumerate(order)}
        assert all(pos[a] < pos[b] for a, b in edges)


def test_tie_break_is_lexicographically_smallest_topological_order():
    # brute force over all permutations (the definition), n <= 7
    rng = np.random.default_rng(11)
    for _ in range(40):
        n = int(rng.integers(1, 8))
        edges = random_dag(rng, n, 0.3)
        valid = [p for p in itertools.permutations(range(n))
                 if all(p.index(a) < p.index(b) for a, b in edges)]
        assert kahn(n, edges) == list(min(valid))


def test_chain_and_no_edges():
    assert kahn(5, [(4, 3), (3, 2), (2, 1), (1, 0)]) == [4, 3, 2, 1, 0]
    assert kahn(4, []) == [0, 1, 2, 3]  # insertion order when nothing constrains
    assert kahn(0, []) == []


@pytest.mark.parametrize("k", [2, 3, 6])
def test_cycles_are_rejected(k):
    g = capi.TaskGraph()
    ids = [g.add(f"c{i}") for i in range(k + 2)]
    g.edge(ids[-1], ids[0])  # an acyclic tail
    for i in range(k):
        g.edge(ids[i], ids[(i + 1) % k])
    with pytest.raises(capi.DPDError) as e:
        g.order()
    assert e.value.code == capi.DPD_ERR_CONFIG


def test_bad_edges():
    g = capi.TaskGraph()
    a = g.add("a")
    for bad in [(a, a), (a, 5), (-1, a)]:
        with pytest.raises(capi.DPDError):
            g.edge(*bad)


def test_writer_depth0_is_synchronous(tmp_path):
    q = capi.IoQueue(0)
    p = tmp_path / "x.bin"
    q.write(str(p), b"abc", delay_us=20000)
    assert p.read_bytes() == b"abc"  # written before write() returned
    assert q.pending() == 0
    assert q.close() == 1


def test_writer_drains_on_close_and_never_drops(tmp_path):
    q = capi.IoQueue(4)
    data = [os.urandom(int(n)) for n in np.random.default_rng(3).integers(0, 5000, 25)]
    for k, d in enumerate(data):
        q.write(str(tmp_path / f"f{k}"), d, delay_us=2000)
    assert q.close() == len(data)
    for k, d in enumerate(data):
        assert (tmp_path / f"f{k}").read_bytes() == d


def test_writer_overlaps_and_applies_backpressure(tmp_path):
    # slow disk: 40 ms per write, depth 2.  The first submissions return at once (overlap);
    # at most depth + 1 (running) are ever outstanding; later ones block (backpressure).
    depth, delay = 2, 0.04
    q = capi.IoQueue(depth)
    t0 = time.perf_counter()
    q.write(str(tmp_path / "a"), b"a", delay_us=int(delay * 1e6))
    t_first = time.perf_counter() - t0
    assert t_first < delay / 2
    seen = []
    for k in range(6):
        q.write(str(tmp_path / f"b{k}"), b"b", delay_us=int(delay * 1e6))
        seen.append(q.pending())
    t_all = time.perf_counter() - t0
    assert max(seen) <= depth + 1
    assert t_all >= 3 * delay  # 7 writes through a 2-deep queue cannot all be accepted at once
    assert q.close() == 7


def test_writer_error_surfaces_at_next_write_or_close(tmp_path):
    bad = str(tmp_path / "no_such_dir" / "x")
    q = capi.IoQueue(2)
    q.write(bad, b"x")
    time.sleep(0.1)  # the worker has failed by now
    with pytest.raises(capi.DPDError) as e:
        q.write(str(tmp_path / "ok"), b"y")
    assert e.value.code == capi.DPD_ERR_IO and "no_such_dir" in str(e.value)
    q.write(str(tmp_path / "ok2"), b"z")  # reported once; the queue keeps working
    assert q.close() == 1  # ok2 only ("ok" was refused, the failed job does not count)
    q2 = capi.IoQueue(2)
    q2.write(bad, b"x")
    with pytest.raises(capi.DPDError):
        q2.close()
