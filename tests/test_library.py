"""CPU checks of the C-ABI library: it is built for sm_100a, loads without a GPU, and exports every
function include/moddit.h declares (no compute calls here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "moddit.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(mod_[a-z_0-9]+)\s*\(", src)
    return sorted(set(names))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for n in ("mod_collect_block_stats", "mod_fit_mixture", "mod_predict_block_mask", "mod_update_online_mask",
              "mod_block_sparse_attn_fwd", "mod_plan_create", "mod_plan_destroy", "mod_last_error"):
        assert n in names


def test_library_loads_and_exports_every_declared_symbol():
    import paper_2601_11641_b200 as m
    lib = ctypes.CDLL(m.LIB_PATH)
    for n in declared_functions():
        assert hasattr(lib, n), f"{n} declared in moddit.h but not exported"
    from paper_2601_11641_b200._lib import SIGNATURES
    assert set(SIGNATURES) == set(declared_functions())


def test_library_is_sm100a_native():
    import paper_2601_11641_b200 as m
    out = subprocess.run(["cuobjdump", "--list-elf", m.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", m.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass        # tcgen05.mma
    assert "UTMALDG" in sass        # TMA loads
    assert "LDTM" in sass and "STTM" in sass   # tcgen05.ld / st


def test_version_and_error_string_without_gpu():
    import paper_2601_11641_b200 as m
    assert b"sm_100a" in m.lib.mod_version()
    from paper_2601_11641_b200._lib import ModLayout, ModConfig
    # invalid layout is rejected on the host before any device work
    h = ctypes.c_void_p()
    st = m.lib.mod_plan_create(ctypes.byref(ModLayout(1, 1, 96, 0, 1, 1, 1, 128)),
                               ctypes.byref(ModConfig(1e-8, 0.0, 1, 0, 0.0, 0, 1, 1, 0.0, 0)), 0, ctypes.byref(h))
    assert st == 2 and b"head_dim=96" in m.lib.mod_last_error()


def test_plain_c_example_links_against_the_library():
    """examples/moddit_step.c drives the hot path through moddit.h alone (no Python); it must build
    and resolve libmoddit.so from the tree (the GPU run is tests/test_gpu_c_example.py)."""
    from paper_2601_11641_b200.build import build_examples
    exe = os.path.join(ROOT, "examples", "moddit_step")
    if not os.path.exists(exe):
        build_examples()
    out = subprocess.run(["ldd", exe], capture_output=True, text=True).stdout
    assert re.search(r"libmoddit\.so => .*paper_2601_11641_b200/libmoddit\.so", out), out
    usage = subprocess.run([exe], capture_output=True, text=True)
    assert usage.returncode == 1 and "usage" in usage.stderr
