"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel totals and shares."""
import collections
import csv
import sys


def main(path, skip_setup=True):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").split("<unnamed>::")[-1].strip()
        v = float(r[vi].replace(",", "")) * {"ns": 1, "nsecond": 1, "usecond": 1e3, "us": 1e3,
                                              "msecond": 1e6}.get(r[ui], 1)
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    print(f"{'kernel':44s} {'launches':>8s} {'total us':>10s} {'share':>6s} {'avg us':>8s}")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k[:44]:44s} {cnt[k]:8d} {v / 1e3:10.1f} {100 * v / T:5.1f}% {v / cnt[k] / 1e3:8.2f}")


if __name__ == "__main__":
    main(sys.argv[1])
