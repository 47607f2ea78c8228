"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
every entry point include/cprand_b200.h declares, and its host-only calls
behave like the reference (no device compute here)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cprand_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(cprand_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_reference_entry_points():
    names = declared_functions()
    for want in ("cprand_solve", "cprand_gather_fibers", "cprand_skr", "cprand_mode_update",
                 "cprand_estimate_fit", "cprand_mix_tensor", "cprand_session_create"):
        assert want in names


def test_library_exports_every_declared_symbol():
    import paper_1701_06600_b200 as pb
    lib = pb.lib()
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert missing == []
    assert set(declared_functions()) == set(pb.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", pb.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    for n in declared_functions():
        assert re.search(rf"\bT {n}$", out, flags=re.M), n


def test_library_is_sm100a():
    import paper_1701_06600_b200 as pb
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", pb.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_options_defaults_mirror_solve_options():
    import paper_1701_06600_b200 as pb
    from paper_1701_06600_b200._lib import Options
    o = Options()
    pb.lib().cprand_options_init(C.byref(o))
    # solver.hpp:41-52
    assert o.max_iters == 200 and o.fit_tolerance == 1e-4 and o.has_fit_threshold == 0
    assert o.rng_seed == 0 and o.init == 0 and o.fit_sample_count == 1 << 14
    assert o.stall_limit == 10 and o.transform == -1
    assert o.bench_mode == o.exhaustive_samples == o.exact_fit_trace == 0


def test_default_sample_count_matches_reference():
    import paper_1701_06600_b200 as pb
    for r, s in [(1, 10), (2, 14), (5, 80), (6, 108)]:  # test_sampling.cpp:25-31
        assert pb.default_sample_count(r) == s
    with pytest.raises(pb.InvalidArgument):
        pb.default_sample_count(0)


def test_no_cpu_fallback_without_device():
    """Without a GPU the product path must fail loudly, never compute on the host."""
    import numpy as np
    import paper_1701_06600_b200 as pb
    if pb.device_count() > 0:
        pytest.skip("a device is visible")
    with pytest.raises(pb.CprandError) as e:
        pb.cprand(np.ones((3, 3, 3)), 1, 2)
    assert e.value.status == 4


def test_cpp_dropin_header_compiles():
    out = os.path.join(ROOT, "build", "dropin_check")
    src = os.path.join(ROOT, "tests", "cpp", "dropin_smoke.cpp")
    subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", os.path.join(ROOT, "include"), src],
                   check=True)
    assert os.path.exists(src) and out


def test_device_check_build_differs_only_by_checks():
    """The device-check variant (make checklib) exports the same C ABI and
    carries the trap messages; the product library has none of them."""
    prod = os.path.join(ROOT, "paper_1701_06600_b200", "libcprand_b200.so")
    chk = os.path.join(ROOT, "paper_1701_06600_b200", "libcprand_b200_check.so")
    if not os.path.exists(chk):
        pytest.skip("device-check library not built (make checklib)")
    data_p, data_c = open(prod, "rb").read(), open(chk, "rb").read()
    assert b"CPB_DCHECK failed" in data_c and b"CPB_DCHECK failed" not in data_p
    sym = lambda p: set(re.findall(r"\bT (cprand_\w+)$", subprocess.run(  # noqa: E731
        ["nm", "-D", "--defined-only", p], capture_output=True, text=True, check=True).stdout, flags=re.M))
    assert sym(prod) == sym(chk) and len(sym(prod)) > 20
