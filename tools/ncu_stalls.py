"""Stall-reason breakdown of a kernel's hot code regions from an ncu report
(source page, SASS view). Development helper.

usage: python tools/ncu_stalls.py REPORT KERNEL_REGEX
"""
import collections
import csv
import io
import subprocess
import sys


def main(rep, kern):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    tot = collections.Counter()
    per_op = collections.Counter()
    H, reasons = None, []
    for r in rows:
        if r and r[0] == "Address":  # header of one launch's table
            if H is not None:
                break  # first launch only
            H = {h: i for i, h in enumerate(r)}
            reasons = [h for h in r if h.startswith("stall_") and "(Not" not in h]
            continue
        if H is None or len(r) < len(H):
            continue
        op = r[1].split()
        if not op:
            continue
        name = op[1] if op[0].startswith("@") else op[0]
        for h in reasons:
            try:
                v = int(r[H[h]] or 0)
            except ValueError:
                continue
            tot[h] += v
            per_op[(name.split(".")[0], h)] += v
    s = sum(tot.values())
    print(f"{kern}: {s} samples")
    for k, v in tot.most_common(10):
        print(f"  {k:28s} {100 * v / s:5.1f}%")
    print("top (opcode, reason):")
    for (op, h), v in per_op.most_common(15):
        print(f"  {op:12s} {h:26s} {100 * v / s:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
