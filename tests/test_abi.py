"""The C-ABI library without a GPU: it loads, exports every function include/mapsq.h declares,
and its host-only join planner derives the spec the paper describes."""
from __future__ import annotations

import os
import re

import pytest

import paper_1702_03484_b200 as mq

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "mapsq.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mapsq_[a-z_]+)\s*\(", src)))


def test_library_loads_and_exports_every_declared_symbol():
    L = mq.lib()
    declared = _declared_functions()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(L, name), f"{name} declared in include/mapsq.h but not exported"
    assert "sm_100a" in mq.version()


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        mq.Context(0)


def test_plan_single_key_p64():
    # Tp1(?person=0, ?job=1) ⋈ Tp2(?job=1): key ?job, Table 1 bounds
    pl = mq.plan_join([0, 1], [(0, 5), (2, 6)], 3, [1], [(4, 6)], 2)
    assert pl.nshared == 1 and pl.shared[0] == 1
    assert [pl.out_var[i] for i in range(pl.out_ncols)] == [1, 0]   # shared ++ Tp1 rest ++ Tp2 rest
    assert pl.key_col1[0] == 1 and pl.key_col2[0] == 0
    # union bounds [2, 6] -> 3 key bits; n = 5 -> ib = 3 (SURVEY App. A traces ib = 3)
    assert (pl.key_lo[0], pl.key_hi[0], pl.key_bits[0]) == (2, 6, 3)
    assert pl.kb == 3 and pl.ib == 3 and pl.path == mq.PATH_P64 and pl.passes == 1


def test_plan_composite_key_order_and_shifts():
    # A = (x=0, z=2, a=1), B = (z=2, x=0, b=3): shared ascending by id -> (0, 2)
    pl = mq.plan_join([0, 2, 1], [(0, 1023), (0, 255), (0, 9)], 100,
                      [2, 0, 3], [(0, 255), (0, 1023), (0, 9)], 50)
    assert [pl.shared[i] for i in range(pl.nshared)] == [0, 2]
    assert [pl.out_var[i] for i in range(pl.out_ncols)] == [0, 2, 1, 3]
    assert [pl.key_bits[i] for i in range(2)] == [10, 8]
    assert [pl.key_shift[i] for i in range(2)] == [8, 0]    # first shared var most significant
    assert pl.kb == 18 and pl.ib == 8 and pl.passes == 3


def test_plan_residual_path_when_key_and_index_exceed_64_bits():
    # two 32-bit key columns + 5 index bits do not fit one word: the wider/first column is
    # packed, the other is checked exactly inside each packed-key group
    R = mq.WIDE_KEY_RESIDUAL
    full = (0, 0xFFFFFFFF)
    pl = mq.plan_join([0, 1], [full, full], 10, [0, 1], [full, full], 10, R)
    assert pl.path == mq.PATH_RESIDUAL and pl.packed_mask == 0b01
    assert pl.kb == 32 and pl.ib == 5 and pl.passes == 4
    # the widest column is packed first, whatever its position
    pl = mq.plan_join([0, 1], [(0, 255), full], 1 << 26, [0, 1], [(0, 255), full], 1 << 26, R)
    assert pl.path == mq.PATH_RESIDUAL and pl.packed_mask == 0b10 and pl.kb == 32
    # 3 columns: the two widest that fit 64 - ib are packed
    pl = mq.plan_join([0, 1, 2], [(0, 2**20), (0, 2**12), (0, 2**24)], 1000,
                      [0, 1, 2], [(0, 2**20), (0, 2**12), (0, 2**24)], 1000, R)
    assert pl.ib == 11 and pl.path == mq.PATH_RESIDUAL and pl.packed_mask == 0b101
    assert pl.kb == 21 + 25


def test_plan_hash_path_is_the_default_for_wide_keys():
    # keys wider than 64 - ib bits, or wider than 32 bits, sort on a 32-bit (or 64 - ib) hash of
    # every shared column; narrower composite keys keep the exact P64 packing
    full = (0, 0xFFFFFFFF)
    pl = mq.plan_join([0, 1], [full, full], 10, [0, 1], [full, full], 10)
    assert pl.path == mq.PATH_HASH and pl.packed_mask == 0 and pl.kb == 32 and pl.passes == 4
    pl = mq.plan_join([0, 1], [full, full], (1 << 31) - 1, [0, 1], [full, full], 1 << 31)
    assert pl.path == mq.PATH_HASH and pl.ib == 32 and pl.kb == 32
    pl = mq.plan_join([0, 1, 2], [(0, 2**20), (0, 2**12), (0, 2**24)], 1000,
                      [0, 1, 2], [(0, 2**20), (0, 2**12), (0, 2**24)], 1000)
    assert pl.path == mq.PATH_HASH and pl.kb == 32          # 59 key bits > 32: hashed
    pl = mq.plan_join([0, 1], [(0, 2**20), (0, 2**10)], 1000, [0, 1], [(0, 2**20), (0, 2**10)], 1)
    assert pl.path == mq.PATH_P64 and pl.kb == 21 + 11      # 32 bits: packed exactly
    with pytest.raises(mq.MapsqError):
        mq.plan_join([0], [(0, 1)], 1, [0], [(0, 1)], 1, 7)


def test_plan_errors():
    with pytest.raises(mq.MapsqError) as e:
        mq.plan_join([0], [(0, 1)], 1, [1], [(0, 1)], 1)
    assert e.value.status == "E_NO_SHARED"
    with pytest.raises(mq.MapsqError) as e:
        mq.plan_join([0], [(0, 1)], 2 ** 31, [0], [(0, 1)], 2 ** 31)
    assert e.value.status == "E_INVALID"
    with pytest.raises(mq.MapsqError) as e:
        mq.plan_join([0, 0], [(0, 1), (0, 1)], 1, [0], [(0, 1)], 1)
    assert e.value.status == "E_INVALID"


def test_plan_disjoint_bounds_flagged():
    pl = mq.plan_join([0], [(0, 10)], 5, [0], [(20, 30)], 5)
    assert pl.disjoint == 1


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_1702_03484_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "import oracle" not in text and "from oracle" not in text
                assert "oracle.h" not in text and "liboracle" not in text
