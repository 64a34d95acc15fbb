"""The reference's own tests and pipeline against the drop-in.

tests/dropin/Makefile builds, from /root/reference's UNMODIFIED sources:

* ``ref_tests_b200``: proj/tests/test_chain_dp.cpp (every DP test case of the
  reference: quantize KATs, the tiny chain, exact schedules, infeasible
  rebuilds, the random_menu property loops against chain_oracle /
  chain_oracle_dijkstra, solve_chain's min-feasible search) and
  proj/tests/test_simulate.cpp, compiled with this repo's include/ first, so
  remat/chain_dp.hpp and remat/simulate.hpp are this repo's and the DP runs
  on the GPU through librkr.so;
* ``ref_simulate_b200``: test_simulate.cpp alone, host only (the replay gate
  of include/remat/simulate.hpp; runs in the CPU suite);
* ``pipeline_b200`` / ``pipeline_gate_b200`` / ``pipeline_ref``:
  tests/dropin/pipeline_check.cpp --
  pipeline.hpp's build_menus (ILP option generation) -> schedule_with_menu
  (solve_chain + the simulate gate) -> flatten_schedule -> chain_max_peak
  over budget ladders -- against the drop-in and against the reference
  alone; the reference's output is the committed golden
  tests/golden/dropin_pipeline.txt.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

BIN = os.path.join(ROOT, "tests", "dropin", "_bin")
GOLDEN = os.path.join(ROOT, "tests", "golden", "dropin_pipeline.txt")


def _bin(name):
    p = os.path.join(BIN, name)
    if not os.path.exists(p):
        pytest.fail(f"{p} not built: run __graft_entry__.build() where /root/reference exists")
    return p


@pytest.mark.gpu
def test_reference_unit_tests_pass_on_the_dropin():
    r = subprocess.run([_bin("ref_tests_b200")], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    # every test case of both files ran (23 TEST_CASEs: 13 in test_chain_dp.cpp, 10 in test_simulate.cpp)
    assert "(0 failed)" in r.stdout and "23 test cases" in r.stdout, r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("binary", ["pipeline_b200", "pipeline_gate_b200"])
def test_reference_pipeline_on_the_dropin_matches_the_reference(binary):
    """pipeline_b200: the reference's pipeline.hpp over this repo's DP and
    simulator; pipeline_gate_b200: this repo's own gate (remat_b200/gate.hpp)."""
    r = subprocess.run([_bin(binary)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    want = open(GOLDEN).read().splitlines()
    got = r.stdout.splitlines()
    assert len(got) == len(want)
    for a, b in zip(got, want):
        assert a == b


def test_dropin_binaries_bind_the_device_library():
    """The drop-in builds call into librkr (not the reference's header-only
    DP); the reference build does not."""
    for name, want in (("ref_tests_b200", True), ("pipeline_b200", True), ("pipeline_gate_b200", True),
                       ("pipeline_ref", False)):
        p = _bin(name)
        syms = subprocess.run(["nm", "-D", p], capture_output=True, text=True).stdout
        assert ("rkr_solve_chain" in syms or "rkr_table_create" in syms) == want, name


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj"), reason="needs /root/reference")
def test_pipeline_golden_regenerates_from_the_reference():
    r = subprocess.run([_bin("pipeline_ref")], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0
    assert r.stdout == open(GOLDEN).read()


def test_reference_simulate_tests_pass_on_this_simulator():
    """The reference's test_simulate.cpp, unchanged, against include/remat/simulate.hpp."""
    r = subprocess.run([_bin("ref_simulate_b200")], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "10 test cases (0 failed)" in r.stdout, r.stdout


def test_parallel_option_generation_equals_the_reference():
    """remat::b200::build_menus (every (class, budget pair) ILP solve on a
    thread pool, the lattice's dependencies kept: include/remat_b200/menus.hpp)
    returns the reference's build_menus MenuSet member for member on its
    random chains (host only)."""
    r = subprocess.run([_bin("menus_check"), "4"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr[-2000:]
    assert "mismatches 0" in r.stdout, r.stdout
