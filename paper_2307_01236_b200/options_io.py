"""On-disk option menus (``kind: "options"``) as the solver's input -- SURVEY
§8(f) rank 3.

Host-side mirror of the reference's file layer for this path:

* ``read_options_file`` / ``write_options_file`` follow ``tools/remat.cpp:72-123``
  (classes of equivalent blocks, each with a representative and members; every
  block must be covered) and ``decode_options`` / ``encode_options``
  (``include/remat/ingest.hpp:409-481``: field names, the optional
  ``time_bwd_us``, block-local ``fwd_ops`` / ``bwd_ops`` whose targets must
  exist in the representative block).
* ``load_chain`` reads the id- and size-bearing part of a ``kind: "chain"``
  document (``ingest.hpp:144-230``): per block the node ids, the input/output
  data nodes and the loss node -- what ``solve_chain`` needs for activation
  sizes (``types.hpp:270-273``) and schedule op ids (``chain_dp.hpp:218-239``).
  The full CD-graph validation (``validate_chain``) belongs to the out-of-scope
  ingest layer and is not repeated.
* Document framing and field checks follow ``read_document`` /
  ``require_fields`` (``ingest.hpp:25-60``): integer ``format_version`` == 1,
  the expected ``kind``, required fields present, unknown fields rejected.

Errors keep the reference's categories: ``IoError`` (cannot open),
``ParseError`` (malformed document), ``rotor.ValidationError`` (a well-formed
document that is inconsistent with the chain).
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import Dict, List, Sequence

from .menu import BlockOption, Menu
from .rotor import Chain, ValidationError

FORMAT_VERSION = 1  # remat::kFormatVersion


class IoError(RuntimeError):
    """remat::IoError: a file cannot be opened."""


class ParseError(RuntimeError):
    """remat::ParseError: a document is not what its kind requires."""


def _require_fields(j, required: Sequence[str], optional: Sequence[str], where: str) -> None:
    # ingest.hpp:25-37
    if not isinstance(j, dict):
        raise ParseError(f"{where}: expected an object")
    for f in required:
        if f not in j:
            raise ParseError(f"{where}: missing field '{f}'")
    for k in j:
        if k not in required and k not in optional:
            raise ParseError(f"{where}: unknown field '{k}'")


def _int(v, where: str) -> int:
    if isinstance(v, bool) or not isinstance(v, int):
        raise ParseError(f"{where}: expected an integer, found {v!r}")
    return v


def read_document(path: str, expected_kind: str) -> dict:
    """ingest.hpp:39-60."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError as e:
        raise IoError(f"cannot open {path}") from e
    try:
        j = json.loads(text)
    except json.JSONDecodeError as e:
        raise ParseError(f"{path}: {e}") from e
    if not isinstance(j, dict):
        raise ParseError(f"{path}: top level must be an object")
    fv = j.get("format_version")
    if isinstance(fv, bool) or not isinstance(fv, int):
        raise ParseError(f"{path}: missing integer format_version")
    if fv != FORMAT_VERSION:
        raise ParseError(f"{path}: unsupported version {fv}")
    if not isinstance(j.get("kind"), str):
        raise ParseError(f"{path}: missing kind")
    if j["kind"] != expected_kind:
        raise ParseError(f"{path}: expected kind '{expected_kind}', found '{j['kind']}'")
    return j


# ---------------------------------------------------------------------------
# chains: the ids and sizes the DP needs
# ---------------------------------------------------------------------------
@dataclass
class BlockIds:
    """The part of a chain block (remat::CDGraph) the chain DP reads."""

    cnodes: List[str]
    dnodes: Dict[str, int]  # id -> size
    input_data: str
    output_data: str
    loss_id: str

    @property
    def input_size(self) -> int:  # types.hpp:97
        return self.dnodes[self.input_data]

    @property
    def output_size(self) -> int:  # types.hpp:98
        return self.dnodes[self.output_data]


@dataclass
class LoadedChain:
    blocks: List[BlockIds]
    equiv_classes: List[int] = field(default_factory=list)

    def length(self) -> int:
        return len(self.blocks)

    def act_size(self, i: int) -> int:
        """a_i (types.hpp:270-273): block i's input size, the last output for i = L."""
        if i < self.length():
            return self.blocks[i].input_size
        return self.blocks[-1].output_size

    def act_sizes(self) -> List[int]:
        return [self.act_size(i) for i in range(self.length() + 1)]

    def chain(self) -> Chain:
        """The id-bearing chain solve_chain's schedule ops refer to."""
        return Chain([b.input_data for b in self.blocks], [b.loss_id for b in self.blocks])


_DNODE_KINDS = ("data", "grad", "phantom")        # ingest.hpp:94-99
_CNODE_KINDS = ("forward", "backward", "loss")    # ingest.hpp:78-83


def _decode_block(jb, where: str) -> BlockIds:
    # ingest.hpp:144-200 (ids, sizes, kinds, references)
    _require_fields(jb, ("cnodes", "dnodes", "input_data", "output_data", "loss_id"), (), where)
    dn: Dict[str, int] = {}
    for jd in jb["dnodes"]:
        _require_fields(jd, ("id", "size", "kind", "parents"), (), where + ".dnodes")
        if jd["kind"] not in _DNODE_KINDS:
            raise ParseError(f"{where}: unknown dnode kind '{jd['kind']}'")
        if jd["id"] in dn:
            raise ValidationError(f"{where}: duplicate dnode id {jd['id']}")
        dn[jd["id"]] = _int(jd["size"], where + ".dnodes.size")
    cn: List[str] = []
    for jc in jb["cnodes"]:
        _require_fields(jc, ("id", "kind", "time_us", "tmp_mem", "deps", "outputs"), (),
                        where + ".cnodes")
        if jc["kind"] not in _CNODE_KINDS:
            raise ParseError(f"{where}: unknown cnode kind '{jc['kind']}'")
        if jc["id"] in cn:
            raise ValidationError(f"{where}: duplicate cnode id {jc['id']}")
        for d in list(jc["deps"]) + list(jc["outputs"]):
            if d not in dn:
                raise ValidationError(f"{where}: cnode {jc['id']} references '{d}', which does not exist")
        cn.append(jc["id"])
    for name, pool in (("input_data", dn), ("output_data", dn), ("loss_id", cn)):
        if jb[name] not in pool:
            raise ValidationError(f"{where}: {name} '{jb[name]}' does not exist")
    return BlockIds(cn, dn, jb["input_data"], jb["output_data"], jb["loss_id"])


def decode_chain(j: dict, where: str) -> LoadedChain:
    """ingest.hpp:216-230."""
    _require_fields(j, ("format_version", "kind", "blocks"), ("equiv_classes",), where)
    blocks = [_decode_block(jb, f"{where}.blocks[{i}]") for i, jb in enumerate(j["blocks"])]
    if "equiv_classes" in j:
        eq = [_int(e, where + ".equiv_classes") for e in j["equiv_classes"]]
    else:
        eq = list(range(len(blocks)))
    if not blocks:
        raise ValidationError(f"{where}: chain has no blocks")
    return LoadedChain(blocks, eq)


def load_chain(path: str) -> LoadedChain:
    return decode_chain(read_document(path, "chain"), path)


# ---------------------------------------------------------------------------
# option menus
# ---------------------------------------------------------------------------
@dataclass
class ClassMenu:
    """remat::ClassMenu: one option menu shared by equivalent blocks."""

    class_id: int
    representative: int
    members: List[int]
    options: List[BlockOption]
    fwd_ops: List[list] = field(default_factory=list)  # per option: [(op, target)]
    bwd_ops: List[list] = field(default_factory=list)


@dataclass
class MenuSet:
    classes: List[ClassMenu]
    menu: Menu


def decode_options(block: BlockIds, arr, where: str):
    """ingest.hpp:439-481: options, plus their block-local op lists."""
    out, fwd, bwd = [], [], []
    for jo in arr:
        _require_fields(jo, ("option_id", "time_fwd_us", "save_mem", "peak_fwd", "peak_fwd_pre",
                             "peak_bwd", "fwd_ops", "bwd_ops"), ("time_bwd_us",), where)
        o = BlockOption(
            option_id=_int(jo["option_id"], where + ".option_id"),
            time_fwd=_int(jo["time_fwd_us"], where + ".time_fwd_us"),
            time_bwd=_int(jo["time_bwd_us"], where + ".time_bwd_us") if "time_bwd_us" in jo else None,
            save_mem=_int(jo["save_mem"], where + ".save_mem"),
            peak_fwd=_int(jo["peak_fwd"], where + ".peak_fwd"),
            peak_fwd_pre=_int(jo["peak_fwd_pre"], where + ".peak_fwd_pre"),
            peak_bwd=_int(jo["peak_bwd"], where + ".peak_bwd"),
        )

        def read(ja):
            ops = []
            for jl in ja:
                _require_fields(jl, ("op", "target"), (), where + ".ops")
                k, target = jl["op"], jl["target"]
                if k == "compute":
                    ok = target in block.cnodes
                elif k == "forget":
                    ok = target in block.dnodes
                else:
                    raise ParseError(f"{where}: unknown local op '{k}'")
                if not ok:
                    raise ValidationError(f"{where}: option references missing node {target}")
                ops.append((k, target))
            return ops

        fwd.append(read(jo["fwd_ops"]))
        bwd.append(read(jo["bwd_ops"]))
        out.append(o)
    return out, fwd, bwd


def read_options_file(chain: LoadedChain, path: str) -> MenuSet:
    """tools/remat.cpp:93-123: every block's menu from its class, act sizes from the chain."""
    j = read_document(path, "options")
    _require_fields(j, ("format_version", "kind", "classes"), (), path)
    L = chain.length()
    class_of_block = [-1] * L
    classes: List[ClassMenu] = []
    for jc in j["classes"]:
        _require_fields(jc, ("class_id", "representative", "members", "options"), (), path)
        c = ClassMenu(_int(jc["class_id"], path), _int(jc["representative"], path),
                      [_int(m, path) for m in jc["members"]], [])
        if c.representative < 0 or c.representative >= L:
            raise ValidationError(f"{path}: representative out of range")
        c.options, c.fwd_ops, c.bwd_ops = decode_options(chain.blocks[c.representative],
                                                         jc["options"], path)
        for m in c.members:
            if m < 0 or m >= L:
                raise ValidationError(f"{path}: member out of range")
            class_of_block[m] = c.class_id
        classes.append(c)
    for i in range(L):
        if class_of_block[i] < 0:
            raise ValidationError(f"{path}: block {i} has no option menu")
        # the reference indexes the class list by class id (remat.cpp:118);
        # an id outside it would be out of bounds there
        if class_of_block[i] >= len(classes):
            raise ValidationError(f"{path}: block {i}: class id {class_of_block[i]} out of range")
    menu = Menu.from_options([classes[class_of_block[i]].options for i in range(L)],
                             chain.act_sizes())
    return MenuSet(classes, menu)


def encode_options(c: ClassMenu) -> list:
    """ingest.hpp:409-437."""
    arr = []
    for q, o in enumerate(c.options):
        jo = {"option_id": o.option_id, "time_fwd_us": o.time_fwd}
        if o.time_bwd is not None:
            jo["time_bwd_us"] = o.time_bwd
        jo.update(save_mem=o.save_mem, peak_fwd=o.peak_fwd, peak_fwd_pre=o.peak_fwd_pre,
                  peak_bwd=o.peak_bwd)
        ops = lambda lst: [{"op": k, "target": t} for k, t in lst]  # noqa: E731
        jo["fwd_ops"] = ops(c.fwd_ops[q] if q < len(c.fwd_ops) else [])
        jo["bwd_ops"] = ops(c.bwd_ops[q] if q < len(c.bwd_ops) else [])
        arr.append(jo)
    return arr


def write_options_file(classes: Sequence[ClassMenu], path: str) -> None:
    """tools/remat.cpp:72-91."""
    j = {"format_version": FORMAT_VERSION, "kind": "options",
         "classes": [{"class_id": c.class_id, "representative": c.representative,
                      "members": list(c.members), "options": encode_options(c)} for c in classes]}
    with open(path, "w") as f:
        json.dump(j, f, indent=2)


def solve_files(chain_path: str, options_path: str, memory: int, units: int = 500,
                device: int = 0):
    """`remat solve chain.json --memory B --load-options opts.json` down to the
    chain DP (tools/remat.cpp:159-166): the device solve_chain on the loaded menu."""
    from .rotor import solve_chain

    chain = load_chain(chain_path)
    ms = read_options_file(chain, options_path)
    return solve_chain(chain.chain(), ms.menu, memory, units, device=device)


def sweep_files(chain_path: str, options_path: str, budgets: Sequence[int], units: int = 500,
                device: int = 0):
    """`remat sweep --load-options` down to the chain DP (tools/remat.cpp:217-263)."""
    from .rotor import sweep

    chain = load_chain(chain_path)
    ms = read_options_file(chain, options_path)
    return sweep(ms.menu, budgets, units, device=device)


def skeleton_chain_document(act_sizes: Sequence[int], loss_time: int = 0) -> dict:
    """A minimal valid ``kind: "chain"`` document with the given activation
    sizes (block i: input ``b{i}_in``, output ``b{i}_out``, loss ``b{i}_loss``):
    the synthetic chains of the tests and benchmarks as files."""
    L = len(act_sizes) - 1
    blocks = []
    for i in range(L):
        blocks.append({
            "cnodes": [
                {"id": f"b{i}_f", "kind": "forward", "time_us": 1, "tmp_mem": 0,
                 "deps": [f"b{i}_in"], "outputs": [f"b{i}_out"]},
                {"id": f"b{i}_loss", "kind": "loss", "time_us": loss_time, "tmp_mem": 0,
                 "deps": [f"b{i}_out"], "outputs": [f"b{i}_g_out"]},
                {"id": f"b{i}_b", "kind": "backward", "time_us": 1, "tmp_mem": 0,
                 "deps": [f"b{i}_g_out", f"b{i}_in"], "outputs": [f"b{i}_g_in"]},
            ],
            "dnodes": [
                {"id": f"b{i}_in", "size": int(act_sizes[i]), "kind": "data", "parents": []},
                {"id": f"b{i}_out", "size": int(act_sizes[i + 1]), "kind": "data",
                 "parents": [f"b{i}_f"]},
                {"id": f"b{i}_g_out", "size": int(act_sizes[i + 1]), "kind": "grad",
                 "parents": [f"b{i}_loss"]},
                {"id": f"b{i}_g_in", "size": int(act_sizes[i]), "kind": "grad",
                 "parents": [f"b{i}_b"]},
            ],
            "input_data": f"b{i}_in", "output_data": f"b{i}_out", "loss_id": f"b{i}_loss",
        })
    return {"format_version": FORMAT_VERSION, "kind": "chain", "blocks": blocks}


def classes_of_menu(menu: Menu) -> List[ClassMenu]:
    """One class per block of an in-memory menu (the writer's input)."""
    out = []
    for i in range(menu.L):
        out.append(ClassMenu(i, i, [i], menu.options(i)))
    return out
