"""Attribute an ncu source-page capture (SASS view) to CUDA source lines.

  ncu -i prof.ncu-rep --page source --csv --print-source sass > k.csv
  python scripts/ncu_lines.py k.csv <mangled kernel name> [metric] [top] [--callsite]

Disassembles the kernel from the built library with line info (nvdisasm -g), maps every
SASS offset to its (file, line), and sums the metric (default: all warp-stall samples) per
source line -- the per-line view the CLI does not print for stripped captures.
"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2011_09208_b200", "lib", "libwhale_splitfc.so")


WRAPPERS = ("ptx_sm100.cuh", ".hpp", ".h")


def sass_lines(kernel, callsite=False):
    """offset -> (file, line); callsite=True attributes inlined PTX wrappers / CUDA headers to
    the first enclosing line in the kernel sources (e.g. WHICH mbar_wait a warp sits in)."""
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", LIB], cwd=d, check=True, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    out = subprocess.run(["nvdisasm", "-gi" if callsite else "-g", "-c", os.path.join(d, cub)], capture_output=True,
                         text=True).stdout
    sec = out[out.index(f".text.{kernel}"):]
    nxt = sec.find("//--------------------- .text.", 10)
    sec = sec[:nxt] if nxt > 0 else sec
    cur = ("?", 0)
    frames = []
    m = {}
    for ln in sec.splitlines():
        if "//## File" in ln:
            frames += [(os.path.basename(f), int(l)) for f, l in re.findall(r'"([^"]+)", line (\d+)', ln)]
            continue
        mo = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if mo:
            if frames:
                cur = frames[0]
                if callsite:
                    cur = next((fr for fr in frames if not fr[0].endswith(WRAPPERS)), frames[-1])
            frames = []
            m[int(mo.group(1), 16)] = cur
    return m


def main():
    path, kernel = sys.argv[1], sys.argv[2]
    metric = sys.argv[3] if len(sys.argv) > 3 else "Warp Stall Sampling (All Samples)"
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    callsite = "--callsite" in sys.argv
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Address" in r)
    hdr = rows[hi]
    idx = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
    base = min(int(r[idx["Address"]], 16) for r in data)
    m = sass_lines(kernel, callsite)
    acc = collections.Counter()
    for r in data:
        off = int(r[idx["Address"]], 16) - base
        try:
            v = float(r[idx[metric]] or 0)
        except ValueError:
            v = 0.0
        acc[m.get(off, ("?", 0))] += v
    tot = sum(acc.values())
    print(f"total {metric}: {tot:.0f}")
    for (f, ln), v in acc.most_common(top):
        print(f"{v:10.0f} {100 * v / max(tot, 1):5.1f}%  {f}:{ln}")


if __name__ == "__main__":
    main()
