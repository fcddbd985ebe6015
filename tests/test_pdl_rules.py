"""The cross-launch overlap rule (csrc/abi.cu pdl_early, reached through the
diagnostics entry dctadj_pdl_probe): a launch may skip its entry wait on the
previous grid of its stream only when its byte ranges overlap none of the
launches that may still be running there -- every launch since the last one
that waited at entry.  Pure host logic: runs without a GPU (stream handles and
buffer addresses are only keys here)."""
import ctypes

import pytest

from paper_2505_23618_b200 import _lib

_next_stream = [0x5000]


def _stream():
    _next_stream[0] += 0x10
    return ctypes.c_void_p(_next_stream[0])


@pytest.fixture(scope="module")
def lib():
    return _lib.load()


def probe(lib, st, src, nsrc, dst, ndst):
    r = lib.dctadj_pdl_probe(st, ctypes.c_void_p(src), nsrc, ctypes.c_void_p(dst), ndst, 0)
    assert r in (0, 1)
    return r == 1


def test_first_launch_waits_then_independent_ones_overlap(lib):
    st = _stream()
    assert not probe(lib, st, 0x10000, 100, 0x20000, 100)   # unknown history
    assert probe(lib, st, 0x30000, 100, 0x40000, 100)       # independent
    assert probe(lib, st, 0x50000, 100, 0x60000, 100)


@pytest.mark.parametrize("src,dst,why", [
    (0x20000, 0x90000, "read after write"),
    (0x90000, 0x10000, "write after read"),
    (0x90000, 0x20050, "write after write"),
    (0x90000, 0x1ffd0, "partial overlap at the start"),
])
def test_dependent_launch_waits(lib, src, dst, why):
    st = _stream()
    assert not probe(lib, st, 0x10000, 100, 0x20000, 100)
    assert not probe(lib, st, src, 100, dst, 100), why


def test_adjacent_ranges_do_not_conflict(lib):
    st = _stream()
    probe(lib, st, 0x10000, 0x100, 0x20000, 0x100)
    assert probe(lib, st, 0x10100, 0x100, 0x20100, 0x100)  # [a, a+n) is half-open


def test_dependence_on_any_live_launch_not_just_the_last(lib):
    st = _stream()
    probe(lib, st, 0x10000, 100, 0x20000, 100)             # A (waits)
    assert probe(lib, st, 0x30000, 100, 0x40000, 100)       # B early: A may still run
    assert not probe(lib, st, 0x20000, 100, 0x50000, 100)   # C reads A's output
    # C waited, so A and B are done before C passes its entry wait: only C is live
    assert probe(lib, st, 0x40000, 100, 0x60000, 100)       # reads B's output: fine now


def test_poison_forces_the_next_launch_to_wait(lib):
    st = _stream()
    probe(lib, st, 0x10000, 100, 0x20000, 100)
    assert lib.dctadj_pdl_probe(st, None, 0, None, 0, 1) == 0
    assert not probe(lib, st, 0x70000, 100, 0x80000, 100)
    assert probe(lib, st, 0x90000, 100, 0xa0000, 100)


def test_streams_are_tracked_separately(lib):
    s1, s2 = _stream(), _stream()
    probe(lib, s1, 0x10000, 100, 0x20000, 100)
    probe(lib, s2, 0x10000, 100, 0x30000, 100)
    assert probe(lib, s1, 0x40000, 100, 0x50000, 100)
    assert probe(lib, s2, 0x60000, 100, 0x70000, 100)


def test_live_list_is_bounded(lib):
    st = _stream()
    probe(lib, st, 0x1000, 16, 0x2000, 16)
    got = [probe(lib, st, 0x100000 + 64 * i, 16, 0x900000 + 64 * i, 16) for i in range(40)]
    assert all(got[:31]) and not got[31]  # 32 live launches at most, then one waits
    assert got[32]
