"""Aggregate an ncu report's warp-stall samples by CUDA source line.

usage: python tools/ncu_lines.py report.ncu-rep [top=30]
Needs a capture with --import-source on and a -lineinfo build.  Prints the
lines with the most samples, their share, the dominant stall reasons and the
source text.
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = csv.reader(io.StringIO(out))
    fname, hdr, cur = None, None, None
    samples = defaultdict(float)
    stalls = defaultdict(lambda: defaultdict(float))
    text = {}
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if r[0] == "Function Name" or hdr is None:
            continue
        if r[0]:
            cur = (fname, int(r[0]))
            text[cur] = r[1].strip()
            continue
        if cur is None or len(r) < len(hdr) or r[2] in ("...", "-"):
            continue
        d = dict(zip(hdr[2:], r[2:]))
        try:
            n = float(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            continue
        samples[cur] += n
        for k, v in d.items():
            if k.startswith("stall_") and "Not Issued" not in k:
                try:
                    stalls[cur][k[6:]] += float(v or 0)
                except ValueError:
                    pass
    tot = sum(samples.values()) or 1.0
    print(f"total samples {tot:.0f}")
    for key, n in sorted(samples.items(), key=lambda kv: -kv[1])[:top]:
        st = sorted(stalls[key].items(), key=lambda kv: -kv[1])[:3]
        sts = " ".join(f"{k}:{v / n:.0%}" for k, v in st if v)
        print(f"{100 * n / tot:5.1f}%  {key[0]}:{key[1]:<5d} [{sts}]  {text.get(key, '')[:90]}")


if __name__ == "__main__":
    main()
