"""Summarise an ncu launch-list CSV (gpu__time_duration.sum per launch): top kernels of the
last `frac` of the launches (the measured step after warm-up)."""
import collections
import csv
import sys


def main(path, frac=0.25, top=16):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    last = data[int(len(data) * (1 - frac)):]
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for d in last:
        unit = d["Metric Unit"]
        v = float(d["Metric Value"].replace(",", "")) * (1e-3 if unit in ("ns", "nsecond") else
                                                         1e3 if unit in ("ms", "msecond") else 1.0)
        k = d["Kernel Name"][:90]
        agg[k][0] += 1
        agg[k][1] += v
        tot += v
    print(f"launches {len(last)}  total {tot:.1f} us (serialised, cold)")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{t:9.1f} us {100 * t / tot:5.1f}%  {c:4d}x  {k}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 0.25)
