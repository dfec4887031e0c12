"""CPU checks of the C-ABI boundary: the library loads, exports every symbol include/energon.h
declares, and rejects bad configurations on the host before touching the device."""
import ctypes
import os
import re

import pytest

from paper_2209_02341_b200 import build, energon

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    build()
    return energon.load_library()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "energon.h")).read()
    return sorted(set(re.findall(r"ENERGON_API\s+[\w\s\*]+?\b(energon_\w+)\s*\(", src)))


def test_header_declares_the_binding_names():
    assert declared_symbols() == sorted(energon.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_status_strings(lib):
    for code, name in energon.STATUS.items():
        assert lib.energon_status_string(code).decode() == name


@pytest.mark.parametrize("field,value,status", [
    ("num_heads", 5, -2),      # 64 % 5 != 0: H != h*d
    ("tp_size", 3, -2),        # 4 heads % 3
    ("tp_rank", 2, -2),        # rank >= tp_size
    ("dtype", 7, -2),
    ("comm", 2, -2),           # neither ENERGON_COMM_NCCL nor ENERGON_COMM_P2P
    ("num_layers", 0, -2),
    ("hidden", 12, -2),        # 12 % 4 == 0 but hidden=12/h=4 -> d=3: shape check
])
def test_init_rejects_bad_config_on_host(lib, field, value, status):
    cfg = energon.make_config(1, 64, 4, 256, 256, 16, 64, dtype="f32", tp_size=2 if field == "tp_rank" else 1)
    setattr(cfg, field, value)
    ctx = ctypes.c_void_p()
    rc = lib.energon_init(ctypes.byref(cfg), None, ctypes.byref(ctx))
    if field == "hidden":
        assert rc == -3  # ENERGON_ERR_SHAPE: head_dim 3 not a multiple of 8
    else:
        assert rc == status
    assert not ctx.value
    assert lib.energon_last_error(None).decode()


def test_tp_without_unique_id_rejected(lib):
    cfg = energon.make_config(1, 64, 4, 256, 256, 16, 64, dtype="f32", tp_size=2)
    ctx = ctypes.c_void_p()
    assert lib.energon_init(ctypes.byref(cfg), None, ctypes.byref(ctx)) == -1


def test_index_maps_validates_lengths_on_host(lib):
    lens = (ctypes.c_int32 * 2)(3, 0)
    dummy = ctypes.c_void_p(16)
    assert lib.energon_index_maps(lens, 2, 4, dummy, dummy, dummy, dummy, None) == -4
    lens = (ctypes.c_int32 * 2)(3, 5)
    assert lib.energon_index_maps(lens, 2, 4, dummy, dummy, dummy, dummy, None) == -4


def test_pmep_plan_paper_example(lib):
    """24 layers, 20 resident -> layers 5, 11, 17, 23 are offloaded."""
    import json
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "spec_examples.json")))["pmep_placement"]
    assert energon.energon_pmep_plan(g["num_layers"], g["resident"]) == g["offloaded"]


@pytest.mark.parametrize("L,resident", [(24, 20), (30, 20), (40, 20), (40, 36), (12, 11), (7, 1), (5, 5)])
def test_pmep_plan_is_even(lib, L, resident):
    """'distributed evenly among those to be held on device': m ascending ids ending at
    L-1, consecutive gaps differ by at most one layer."""
    out = energon.energon_pmep_plan(L, resident)
    m = L - resident
    assert len(out) == m and out == sorted(set(out)) and all(0 <= x < L for x in out)
    if m:
        assert out[-1] == L - 1
        gaps = [b - a for a, b in zip([-1] + out[:-1], out)]
        assert max(gaps) - min(gaps) <= 1


def test_pmep_plan_rejects_bad_arguments(lib):
    n = (ctypes.c_int32 * 4)()
    assert lib.energon_pmep_plan(4, 0, n) == -1
    assert lib.energon_pmep_plan(4, 5, n) == -1


def test_stage_plan_paper_example(lib):
    """12 layers on 4 devices -> 3 layers each; SPEC.md:362-367 remainder rule."""
    import json
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "spec_examples.json")))["stage_plan"]
    for ex in g["examples"]:
        assert energon.energon_stage_plan(ex["num_layers"], ex["pp_size"]) == [tuple(r) for r in ex["ranges"]]


@pytest.mark.parametrize("L,pp", [(40, 8), (40, 3), (48, 5), (64, 7), (2, 2), (1, 1)])
def test_stage_plan_partitions(lib, L, pp):
    """Contiguous ranges that partition [0, L), non-empty, sizes differ by at most one, earlier stages larger."""
    r = energon.energon_stage_plan(L, pp)
    assert r[0][0] == 0 and r[-1][1] == L and all(a[1] == b[0] for a, b in zip(r, r[1:]))
    sizes = [e - b for b, e in r]
    assert min(sizes) >= 1 and max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)


def test_stage_plan_rejects_bad_arguments(lib):
    out = (ctypes.c_int32 * 8)()
    assert lib.energon_stage_plan(4, 5, out) == -2
    assert lib.energon_stage_plan(4, 0, out) == -2
    assert lib.energon_stage_plan(4, 2, None) == -1
