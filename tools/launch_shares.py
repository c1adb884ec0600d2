"""Kernel shares of an ncu launch list (--metrics gpu__time_duration.sum --csv):
    python tools/launch_shares.py LAUNCHES.csv [--only-hg]
Per kernel: launches, total and mean duration, share of the listed time.  ncu serialises the
launches (cold caches, no concurrency), so compare SHARES with the live run, not absolute times."""
import collections
import csv
import sys

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def shares(path, only_hg=False):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[vi] == "":
            continue
        name = r[ki].split("(")[0]
        if only_hg and "hg::" not in name:
            continue
        tot[name] += float(r[vi].replace(",", "")) * UNIT[r[ui]]
        cnt[name] += 1
    return tot, cnt


if __name__ == "__main__":
    tot, cnt = shares(sys.argv[1], "--only-hg" in sys.argv)
    T = sum(tot.values())
    print(f"{sum(cnt.values())} launches, {T / 1e3:.1f} ms listed")
    print("| kernel | launches | total ms | share | mean us |")
    print("|---|---|---|---|---|")
    for k, v in tot.most_common(15):
        print(f"| `{k[:90]}` | {cnt[k]} | {v / 1e3:.1f} | {v / T:.3f} | {v / cnt[k]:.1f} |")
