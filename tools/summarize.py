"""Summaries of bench JSON lines and ncu launch lists (used for profiles/)."""
import collections
import csv
import json
import sys


def bench(path):
    d = json.loads(open(path).read().strip().splitlines()[-1])
    print(f"{path}: value {d['value']:.0f} {d['unit']}  ms/step {d['ms_per_step']:.4f}  ns/day/system "
          f"{d['ns_per_day_per_system']:.1f}  launches {d['gpu_launches']}  clocks {d['clocks']}")
    for k, v in d["kernels"].items():
        print("   %-10s %8.4f ms/launch  share %5.3f  %s" % (k, v["ms_per_launch"], v["share_of_step"] or 0,
              f"{v.get('achieved', 0):.1f} {v.get('unit', '')} frac {v.get('frac', 0):.3f}" if 'achieved' in v else ""))


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v = v / 1000.0 if r[ui] in ("ns", "nsecond") else (v * 1000.0 if r[ui] in ("ms", "msecond") else v)
        a = agg.setdefault(r[ki].split("(")[0][:70], [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{n:5d} {t:10.1f} us {t / n:9.2f} us/launch {100 * t / tot:5.1f}%  {k}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        (bench if p.endswith(".json") else launches)(p)
