#!/usr/bin/env python
"""Attribute stall samples and executed instructions of one kernel to CUDA source lines
(ncu --page source --print-source cuda,sass), top N lines.

  python scripts/ncu_lines.py gpurun_out/prof.ncu-rep k_query [N]
"""
import collections
import csv
import io
import subprocess
import sys


def main(rep: str, kre: str, n: int = 40) -> None:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "-k", "regex:" + kre], capture_output=True, text=True).stdout
    samples = collections.Counter()
    execd = collections.Counter()
    text = {}
    fp = "?"
    cur = None
    hdr = None
    seen_fn = set()
    for r in csv.reader(io.StringIO(raw)):
        if not r:
            continue
        if r[0] == "File Path":
            fp = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            if r[1] in seen_fn and fp == "?":
                break
            seen_fn.add(r[1])
            continue
        if r[0] == "Line No":
            hdr = r
            ci, ie = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
            continue
        if hdr is None:
            continue
        if r[0]:
            cur = (fp, int(r[0]))
            text[cur] = r[1].strip()[:90]
        elif cur is not None:
            try:
                samples[cur] += float(r[ci] or 0)
                execd[cur] += int(r[ie] or 0)
            except ValueError:
                pass
    tot = sum(samples.values()) or 1
    print(f"total samples {tot:.0f}")
    for k, v in samples.most_common(n):
        print(f"{v / tot * 100:5.1f}%  ex={execd[k]:>10}  {k[0]}:{k[1]}  {text[k]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
