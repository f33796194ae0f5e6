#!/usr/bin/env python
"""Per-source-line and per-opcode instruction counts of one kernel from an ncu --set full capture
(--import-source on, -lineinfo build), normalised per warp of output points.

    python tools/ncu_source_summary.py gpurun_out/r2_slpipe.ncu-rep 16777216 [top]
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep, npts = sys.argv[1], float(sys.argv[2])
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    W = npts / 32.0
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    cur, per_line, per_op = None, collections.Counter(), collections.Counter()
    line_ops = collections.defaultdict(collections.Counter)
    for r in rows:
        if len(r) < 8 or r[0] == "Line No":
            continue
        if r[0] != "":
            try:
                cur = (int(r[0]), r[1].strip()[:70])
            except ValueError:
                cur = None
            continue
        if cur is None:
            continue
        try:
            n = int(r[7])
        except ValueError:
            continue
        tok = r[3].strip().split()
        if not tok:
            continue
        op = (tok[1] if tok[0].startswith("@") else tok[0]).split(".")[0]
        per_line[cur] += n
        per_op[op] += n
        line_ops[cur][op] += n
    # opcode totals from the SASS-only view (the interleaved view lists inlined SASS under every
    # source line it belongs to, so its sums over-count)
    sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                          capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(sass)))
    hdr = next(r for r in srows if "Instructions Executed" in r)
    iE, iS = hdr.index("Instructions Executed"), hdr.index("Source")
    per_op = collections.Counter()
    for r in srows[srows.index(hdr) + 1:]:
        try:
            n = int(r[iE])
        except (ValueError, IndexError):
            continue
        tok = r[iS].strip().split()
        if tok:
            per_op[(tok[1] if tok[0].startswith("@") else tok[0]).split(".")[0]] += n
    tot = sum(per_op.values())
    print(f"{rep}: {tot / W:.1f} warp instructions per warp of points ({npts:.0f} points)")
    print("per opcode (SASS view):")
    for op, n in per_op.most_common(20):
        print(f"  {op:10s} {n / W:7.1f}")
    print("per source line (interleaved view; inlined SASS is listed under each line it maps to):")
    for (ln, src), n in per_line.most_common(top):
        ops = ", ".join(f"{k}:{v / W:.1f}" for k, v in line_ops[(ln, src)].most_common(4))
        print(f"  {n / W:7.1f}  {ln:4d}  {src:70s} | {ops}")


if __name__ == "__main__":
    main()
