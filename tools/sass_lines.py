"""Per-source-line SASS instruction counts of one kernel (static, not executed).

    python tools/sass_lines.py <cubin> <kernel-substring> [--file rkr_tiles.cu] [--lines 190-240]
    python tools/sass_lines.py <cubin> <kernel-substring> --dump 190-240

Runs `nvdisasm -g -c` (the cubin must be built with -lineinfo), attributes
every instruction to the `//## File ..., line N` marker before it, and prints
the instruction count and opcode mix per source line -- the evidence for
"instructions per candidate" claims about an inner loop.  --dump prints the
instructions of a line range in program order.
"""
from __future__ import annotations

import argparse
import collections
import re
import subprocess
import sys

LINE = re.compile(r'//## File "([^"]+)", line (\d+)')
LABEL = re.compile(r"^(\.L_x_\d+):")
TARGET = re.compile(r"`\((\.L_x_\d+)\)")
INSN = re.compile(r"^\s*/\*([0-9a-f]{4,})\*/\s+(.*?);")


def parse(cubin: str, kern: str):
    out = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True, check=True).stdout
    cur_file, cur_line, inside = None, None, False
    rows, labels, pending = [], {}, []
    for ln in out.splitlines():
        if ln.startswith(".text.") and ln.rstrip().endswith(":"):
            inside = kern in ln
            continue
        if not inside:
            continue
        m = LABEL.match(ln)
        if m:
            pending.append(m.group(1))
            continue
        m = LINE.search(ln)
        if m:
            cur_file, cur_line = m.group(1).rsplit("/", 1)[-1], int(m.group(2))
            continue
        m = INSN.match(ln)
        if m:
            text = m.group(2).strip()
            op = text.split()[1] if text.startswith("@") else text.split()[0]
            addr = int(m.group(1), 16)
            for lb in pending:
                labels[lb] = addr
            pending = []
            rows.append((cur_file, cur_line, addr, op, text))
    parse.labels = labels
    return rows


def loops(rows, min_loads=1):
    """Innermost-first list of backward branches: (start, end, insns, LDG, lines)."""
    out = []
    for f, l, addr, op, text in rows:
        m = TARGET.search(text)
        if op.startswith("BRA") and m and parse.labels.get(m.group(1), 1 << 40) < addr:
            t = parse.labels[m.group(1)]
            body = [r for r in rows if t <= r[2] <= addr]
            nld = sum(1 for r in body if r[3].startswith("LDG"))
            if nld >= min_loads:
                src = sorted({r[1] for r in body if r[0] == f and r[1] is not None})
                out.append((t, addr, len(body), nld, src))
    return sorted(out, key=lambda x: x[2])


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("cubin")
    ap.add_argument("kernel")
    ap.add_argument("--file", default=None)
    ap.add_argument("--lines", default=None)
    ap.add_argument("--dump", default=None)
    ap.add_argument("--loops", action="store_true", help="list loops with >= 4 global loads")
    a = ap.parse_args()
    rows = parse(a.cubin, a.kernel)
    if not rows:
        print("no instructions found for", a.kernel, file=sys.stderr)
        return 1
    if a.loops:
        for t, e, n, nld, src in loops(rows, 4):
            print(f"loop {t:05x}-{e:05x}: {n:4d} insns {nld:3d} LDG  src lines {src[0] if src else '?'}-{src[-1] if src else '?'}")
        return 0
    if a.dump:
        lo, hi = map(int, a.dump.split("-"))
        for f, l, addr, op, text in rows:
            if (a.file is None or f == a.file) and l is not None and lo <= l <= hi:
                print(f"{f}:{l:<5d} {addr:06x}  {text}")
        return 0
    lo, hi = (map(int, a.lines.split("-")) if a.lines else (0, 1 << 30))
    per = collections.defaultdict(collections.Counter)
    for f, l, _, op, _ in rows:
        if (a.file is None or f == a.file) and l is not None and lo <= l <= hi:
            per[(f, l)][op.split(".")[0]] += 1
    tot = 0
    for (f, l), c in sorted(per.items()):
        n = sum(c.values())
        tot += n
        print(f"{f}:{l:<5d} {n:4d}  " + " ".join(f"{k}x{v}" for k, v in c.most_common()))
    print(f"total {tot} instructions in range")
    return 0


if __name__ == "__main__":
    sys.exit(main())
