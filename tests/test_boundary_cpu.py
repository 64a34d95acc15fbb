"""The C-ABI boundary without a GPU: library loads, exports every declared
symbol, host-only entry points behave like the reference, and compute calls
fail loudly (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_2307_01236_b200 import rotor
from paper_2307_01236_b200.menu import tiny_chain_menu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rkr.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(rkr_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = rotor.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.rkr_abi_version() == 2


def test_quantize_matches_reference(kat):
    for b, u, st, unit, bu in kat["quantize"]:
        if st:
            with pytest.raises(rotor.ValidationError):
                rotor.quantize(b, u)
        else:
            q = rotor.quantize(b, u)
            assert (q.unit, q.budget_units) == (unit, bu)
    assert [rotor.to_units(x, 100) for x in (100, 250, 300)] == [1, 3, 3]


def _has_gpu():
    return rotor.lib().rkr_device_ok(0) == 1


def test_no_cpu_fallback():
    if _has_gpu():
        pytest.skip("GPU present: covered by the gpu suite")
    with pytest.raises(rotor.DeviceError):
        rotor.DpTable(tiny_chain_menu(), 1, 12)
    with pytest.raises(rotor.DeviceError):
        rotor.solve_chain(rotor.Chain.skeleton(2), tiny_chain_menu(), 16, 16)


def test_validation_precedes_device():
    """Malformed menus raise ValidationError like the reference, even before
    any device work (chain_dp.hpp:58, :83-85, :94)."""
    m = tiny_chain_menu()
    bad = tiny_chain_menu()
    bad.has_bwd[1] = 0
    with pytest.raises(rotor.ValidationError, match="without a backward"):
        rotor.DpTable(bad, 1, 8)
    nozero = tiny_chain_menu()
    nozero.option_id[2] = 5  # block 1's option 0 becomes a saved option 5
    nozero.has_bwd[2] = 1
    with pytest.raises(rotor.ValidationError, match="lacks option 0"):
        rotor.DpTable(nozero, 1, 8)
    with pytest.raises(rotor.ValidationError):
        rotor.DpTable(m, 1, -1)


def test_cpp_header_compiles():
    src = os.path.join(ROOT, "tests", "cpp", "test_chain_dp_b200.cpp")
    subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", os.path.join(ROOT, "include"), src],
                   check=True)


def test_standalone_headers_compile(tmp_path):
    """Without the reference tree on the include path, the drop-in headers
    (remat/chain_dp.hpp, remat/simulate.hpp) and the gate fall back to the
    standalone vocabulary in include/remat_b200/ and still compile."""
    src = tmp_path / "t.cpp"
    src.write_text('#include "remat_b200/chain_dp.hpp"\n#include "remat_b200/gate.hpp"\n'
                   "int main() { remat::CDGraph g; auto c = remat::single_block_chain(g);"
                   " (void)c; return 0; }\n")
    subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", os.path.join(ROOT, "include"), str(src)],
                   check=True)


def test_cpp_test_binary_links():
    from paper_2307_01236_b200.build import build_cpp_tests

    path = build_cpp_tests()
    out = subprocess.run(["ldd", path], capture_output=True, text=True).stdout
    assert "librkr.so" in out and "not found" not in out.split("librkr.so")[1].split("\n")[0]


def test_replay_gate_matches_reference_model(orc, synthetic):
    """rkr_replay (product, host) == the oracle's replay of the reference model."""
    from paper_2307_01236_b200.menu import synthetic_menu

    for e in synthetic["solves"]:
        if e["status"] != 0:
            continue
        menu = synthetic_menu(e["L"], e["B"], e["M"], e["seed"], byte_scale=e["byte_scale"])
        st, ops, *_ = orc.solve_chain(menu, e["budget"], e["units"])
        assert rotor.replay(menu, ops) == (e["replay_peak"], e["replay_time"])
    m = tiny_chain_menu()
    good = [(2, 0, 1), (2, 1, 1), (0, 1, -1), (3, 1, 1), (3, 0, 1)]
    assert rotor.replay(m, good) == orc.atomic_replay(m, good)
    with pytest.raises(rotor.ValidationError, match="op 1"):
        rotor.replay(m, [(2, 0, 1), (3, 0, 1)])
