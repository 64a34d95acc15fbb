"""On-disk option menus as the solver's input (paper_2307_01236_b200.options_io):
document framing and field checks like the reference's ingest layer
(ingest.hpp:25-60, :409-481; tools/remat.cpp:72-123), round trips, class
sharing, and -- on the GPU -- solve / sweep from files equal to the oracle."""
import json

import numpy as np
import pytest

from paper_2307_01236_b200 import options_io as oio
from paper_2307_01236_b200 import rotor
from paper_2307_01236_b200.menu import synthetic_menu, tiny_chain_menu


def _files(tmp_path, menu, classes=None):
    chain = tmp_path / "chain.json"
    opts = tmp_path / "opts.json"
    chain.write_text(json.dumps(oio.skeleton_chain_document(list(menu.act_sizes))))
    oio.write_options_file(classes or oio.classes_of_menu(menu), str(opts))
    return str(chain), str(opts)


def _same_menu(a, b):
    for f in ("option_offsets", "option_id", "time_fwd", "time_bwd", "has_bwd", "save_mem",
              "peak_fwd", "peak_fwd_pre", "peak_bwd", "act_sizes"):
        np.testing.assert_array_equal(getattr(a, f), getattr(b, f), err_msg=f)


@pytest.mark.parametrize("menu", [tiny_chain_menu(), synthetic_menu(9, 4, 200, 3),
                                  synthetic_menu(5, 2, 80, 11, tie_stress=True)])
def test_round_trip(tmp_path, menu):
    c, o = _files(tmp_path, menu)
    chain = oio.load_chain(c)
    assert chain.length() == menu.L and chain.act_sizes() == list(menu.act_sizes)
    ms = oio.read_options_file(chain, o)
    _same_menu(ms.menu, menu)
    assert chain.chain().input_ids[0] == "b0_in" and chain.chain().loss_ids[-1] == f"b{menu.L - 1}_loss"


def test_classes_share_one_menu(tmp_path):
    menu = synthetic_menu(6, 3, 100, 4)
    # blocks 0, 2, 4 use block 0's options; 1, 3, 5 use block 1's
    cls = [oio.ClassMenu(0, 0, [0, 2, 4], menu.options(0)), oio.ClassMenu(1, 1, [1, 3, 5], menu.options(1))]
    c, o = _files(tmp_path, menu, cls)
    ms = oio.read_options_file(oio.load_chain(c), o)
    for i in range(6):
        assert ms.menu.options(i) == menu.options(i % 2)
    np.testing.assert_array_equal(ms.menu.act_sizes, menu.act_sizes)


def test_block_local_ops_are_checked(tmp_path):
    menu = synthetic_menu(2, 1, 40, 5)
    cls = oio.classes_of_menu(menu)
    cls[0].fwd_ops = [[("compute", "b0_f"), ("forget", "b0_out")] for _ in cls[0].options]
    cls[0].bwd_ops = [[("compute", "b0_b")] for _ in cls[0].options]
    c, o = _files(tmp_path, menu, cls)
    ms = oio.read_options_file(oio.load_chain(c), o)
    assert ms.classes[0].fwd_ops[0] == [("compute", "b0_f"), ("forget", "b0_out")]
    doc = json.loads(open(o).read())
    doc["classes"][0]["options"][0]["fwd_ops"][0]["target"] = "b9_nowhere"
    open(o, "w").write(json.dumps(doc))
    with pytest.raises(rotor.ValidationError, match="missing node"):
        oio.read_options_file(oio.load_chain(c), o)
    doc["classes"][0]["options"][0]["fwd_ops"][0] = {"op": "fold", "target": "b0_f"}
    open(o, "w").write(json.dumps(doc))
    with pytest.raises(oio.ParseError, match="unknown local op"):
        oio.read_options_file(oio.load_chain(c), o)


def _mutate(tmp_path, fn):
    menu = synthetic_menu(3, 2, 60, 6)
    c, o = _files(tmp_path, menu)
    doc = json.loads(open(o).read())
    fn(doc)
    open(o, "w").write(json.dumps(doc))
    return oio.load_chain(c), o


@pytest.mark.parametrize("fn,err,msg", [
    (lambda d: d.update(kind="chain"), oio.ParseError, "expected kind 'options'"),
    (lambda d: d.update(format_version=2), oio.ParseError, "unsupported version"),
    (lambda d: d.pop("format_version"), oio.ParseError, "format_version"),
    (lambda d: d.update(extra=1), oio.ParseError, "unknown field 'extra'"),
    (lambda d: d["classes"][0].pop("members"), oio.ParseError, "missing field 'members'"),
    (lambda d: d["classes"][0]["options"][0].pop("peak_bwd"), oio.ParseError, "missing field 'peak_bwd'"),
    (lambda d: d["classes"][0]["options"][0].update(time_fwd_us=1.5), oio.ParseError, "integer"),
    (lambda d: d["classes"][1].update(members=[7]), rotor.ValidationError, "member out of range"),
    (lambda d: d["classes"][1].update(representative=-1), rotor.ValidationError, "representative"),
    (lambda d: d["classes"].pop(2), rotor.ValidationError, "block 2 has no option menu"),
])
def test_malformed_options_files(tmp_path, fn, err, msg):
    chain, o = _mutate(tmp_path, fn)
    with pytest.raises(err, match=msg):
        oio.read_options_file(chain, o)


def test_chain_document_checks(tmp_path):
    with pytest.raises(oio.IoError):
        oio.load_chain(str(tmp_path / "missing.json"))
    p = tmp_path / "c.json"
    p.write_text("{not json")
    with pytest.raises(oio.ParseError):
        oio.load_chain(str(p))
    doc = oio.skeleton_chain_document([4, 5, 6])
    doc["blocks"][1]["loss_id"] = "nope"
    p.write_text(json.dumps(doc))
    with pytest.raises(rotor.ValidationError, match="loss_id"):
        oio.load_chain(str(p))
    doc = oio.skeleton_chain_document([4, 5, 6])
    doc["blocks"][0]["dnodes"][0]["kind"] = "weird"
    p.write_text(json.dumps(doc))
    with pytest.raises(oio.ParseError, match="unknown dnode kind"):
        oio.load_chain(str(p))


@pytest.mark.gpu
@pytest.mark.parametrize("L,B,M,seed,budget_frac", [(12, 5, 300, 3, 0.6), (24, 8, 500, 41, 0.3)])
def test_solve_and_sweep_from_files(tmp_path, orc, L, B, M, seed, budget_frac):
    menu = synthetic_menu(L, B, M, seed, byte_scale=64)
    c, o = _files(tmp_path, menu)
    peak = int(menu.act_sizes.sum() + menu.peak_fwd.max() * L)
    budget = int(peak * budget_frac)
    st, ref_ops, ref_t, ref_u, ref_mt, ref_mf = orc.solve_chain(menu, budget, 500)
    if st == 0:
        sol = oio.solve_files(c, o, budget, 500)
        assert (sol.opt_time, sol.unit, sol.m_top) == (ref_t, ref_u, ref_mt)
        assert sol.raw_ops == ref_ops
        ids = {f"b{i}_in" for i in range(L)} | {f"b{i}_loss" for i in range(L)}
        assert all(op.target in ids for op in sol.schedule if op.target)
    else:
        with pytest.raises(rotor.InfeasibleBudget) as e:
            oio.solve_files(c, o, budget, 500)
        assert e.value.min_feasible_budget == ref_mf
    rows = oio.sweep_files(c, o, [budget, budget * 2, peak], 500)
    for r in rows:
        st, ops, t, u, mt, mf = orc.solve_chain(menu, r.budget, 500)
        assert r.feasible == (st == 0)
        if st == 0:
            assert (r.opt_time, r.ops) == (t, ops)


# ---------------------------------------------------------------------------
# Documents produced by the reference itself (tests/dropin/options_ref.cpp,
# built against /root/reference alone by tests/dropin/Makefile): its chain
# fixtures proj/tests/fixtures/{tiny,ababab}_chain.json re-encoded by
# ingest.hpp's save_chain, the option menus its ILP generates encoded by
# ingest.hpp's encode_options (the `remat solve --save-options` document), and
# cmd_solve's results (schedule_with_menu) over a budget ladder.
# ---------------------------------------------------------------------------
import os  # noqa: E402

_GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
_REF_FIXTURES = ("tiny", "ababab")
_KIND = {"compute": 0, "forget": 1, "block_fwd": 2, "block_bwd": 3}


def _ref_paths(name):
    return (os.path.join(_GOLD, f"ref_chain_{name}.json"),
            os.path.join(_GOLD, f"ref_options_{name}.json"),
            os.path.join(_GOLD, f"ref_solve_{name}.json"))


@pytest.mark.parametrize("name", _REF_FIXTURES)
def test_reference_encoded_documents_round_trip(tmp_path, name):
    """options_io reads the reference's own documents and writes them back
    with the same content (field for field, option for option)."""
    cpath, opath, _ = _ref_paths(name)
    chain = oio.load_chain(cpath)
    ms = oio.read_options_file(chain, opath)
    out = tmp_path / "again.json"
    oio.write_options_file(ms.classes, str(out))
    assert json.load(open(out)) == json.load(open(opath))
    assert ms.menu.L == chain.length()


@pytest.mark.gpu
@pytest.mark.parametrize("name", _REF_FIXTURES)
def test_reference_options_solve_like_cmd_solve(name):
    """`remat solve --load-options` on the reference's documents: every
    budget's opt_time and block-level schedule (or the min-feasible budget)
    equals the reference's cmd_solve on the same chain and menus.  For the
    tiny chain at 300 B: 86 us."""
    cpath, opath, spath = _ref_paths(name)
    res = json.load(open(spath))
    for row in res["rows"]:
        b = row["budget"]
        if row.get("infeasible"):
            with pytest.raises(rotor.InfeasibleBudget) as e:
                oio.solve_files(cpath, opath, b, res["units"])
            assert e.value.min_feasible_budget == row["min_feasible"], b
            continue
        sol = oio.solve_files(cpath, opath, b, res["units"])
        assert sol.opt_time == row["opt_time"], b
        got = [(o.kind, o.block, o.option, o.target) for o in sol.schedule]
        want = [(_KIND[k], blk, opt, tgt) for k, blk, opt, tgt in row["ops"]]
        assert got == want, b
    if name == "tiny":
        r300 = [r for r in res["rows"] if r["budget"] == 300][0]
        assert r300["opt_time"] == 86 and r300["peak"] == 288
