"""Build-time guard of the ordered ranking (CPU: cuobjdump on the built libahs.so; VERDICT r1 #6,
ADVICE r1).  K6 (onesweep.cuh, RANK = kRankOrdered) and K9r (segsort.cuh, ORD = true) take a key's
stable rank from the old value returned by one shared-memory atomicAdd, which is correct only
because the lanes of one such instruction are served in lane order; k_lane_order_selftest checks
that property on the device before the library selects the ordered kernels.  The self-test only
vouches for the instruction form it executes, so this test asserts that every return-valued
shared atomic in the ordered kernels is the same `ATOMS.ADD Rd, [..], Rs` form as the self-test's
(a toolchain that, say, aggregated the rank atomics into another instruction would fail here), and
that the unordered (masked) kernels never depend on a returned rank this way."""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2506_20677_b200", "lib", "libahs.so")

RE_FUNC = re.compile(r"Function : (\S+)")
RE_ATOMS = re.compile(r"(?:@!?U?P\w+\s+)?(ATOMS\.[A-Z0-9.]+)\s+(\w+),\s*\[([^\]]*)\],?\s*([^;]*);")
RE_K6 = re.compile(r"_ZN3ahs10k_onesweepILb(\d)ELi(\d+)ELi(\d+)ELi(\d+)ELi(\d)E")
RE_K9R = re.compile(r"_ZN3ahs11k_seg_radixI[jm]Lb(\d)ELi(\d+)ELi(\d+)ELb(\d)E")
RE_K6V2 = re.compile(r"_ZN3ahs11k_onesweep2I")  # K6 v2 (onesweep2.cuh): ordered ranking only


@pytest.fixture(scope="module")
def sass():
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(LIB):
        from paper_2506_20677_b200 import build
        build.build()
    out = subprocess.run([cuobjdump, "-sass", LIB], capture_output=True, text=True, check=True).stdout
    funcs, cur = {}, None
    for ln in out.splitlines():
        m = RE_FUNC.search(ln)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            continue
        m = RE_ATOMS.search(ln)
        if m and cur:
            funcs[cur].append((m.group(1), m.group(2)))
    return funcs


def returning(insts):
    """shared atomics whose old value lands in a register (the rank sites)"""
    return [(op, dst) for op, dst in insts if dst != "RZ"]


def ordered_kernels(funcs):
    out = {}
    for f, insts in funcs.items():
        m = RE_K6.search(f)
        if m and m.group(5) == "1":
            out[f] = insts
        m = RE_K9R.search(f)
        if m and m.group(4) == "1":
            out[f] = insts
        if RE_K6V2.search(f):
            out[f] = insts
    return out


def test_selftest_executes_the_plain_returning_atomic(sass):
    st = [f for f in sass if "k_lane_order_selftest" in f]
    assert len(st) == 1
    ret = returning(sass[st[0]])
    assert ret and all(op == "ATOMS.ADD" and re.fullmatch(r"R\d+", dst) for op, dst in ret), ret


def test_ordered_rank_sites_match_the_selftest_form(sass):
    ordered = ordered_kernels(sass)
    # every ordered instantiation the library ships: K6 32/64-bit keys, pairs, 64-bit values; K9r
    assert sum(1 for f in ordered if "k_onesweep" in f) >= 6
    assert sum(1 for f in ordered if "k_seg_radix" in f) >= 8
    assert sum(1 for f in ordered if "k_onesweep2" in f) >= 2  # RADIX keys and pairs
    for f, insts in ordered.items():
        ret = returning(insts)
        assert ret, f"{f}: no returning shared atomic (rank site) found"
        bad = [(op, dst) for op, dst in ret if op != "ATOMS.ADD" or not re.fullmatch(r"R\d+", dst)]
        assert not bad, f"{f}: rank sites compiled to a form the self-test does not execute: {bad}"


def test_masked_kernels_do_not_rank_by_returned_order(sass):
    for f, insts in sass.items():
        m6, m9 = RE_K6.search(f), RE_K9R.search(f)
        if (m6 and m6.group(5) == "0") or (m9 and m9.group(4) == "0"):
            assert not returning(insts), f"{f}: unordered kernel uses a returned shared atomic"
