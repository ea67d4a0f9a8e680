"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ launch__grid_size]):
one line per launch (id, kernel, grid, us) or, with --sum, per kernel name."""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    summ = "--sum" in sys.argv
    rows = list(csv.reader(open(path)))
    hdr, launch = None, collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            e = launch.setdefault(d["ID"], {"name": d["Kernel Name"]})
            e[d["Metric Name"]] = d["Metric Value"].replace(",", "")
    if summ or "--md" in sys.argv:
        tot = collections.defaultdict(lambda: [0, 0.0])
        for v in launch.values():
            t = tot[v["name"].split("(")[0]]
            t[0] += 1
            t[1] += float(v.get("gpu__time_duration.sum", 0)) / 1e3
        allus = sum(us for _, us in tot.values())
        if "--md" in sys.argv:
            print(f"Total {len(launch)} launches, {allus / 1e3:.1f} ms GPU time.\n")
            print("| share | launches | avg us | kernel |\n|---:|---:|---:|---|")
            for k, (n, us) in sorted(tot.items(), key=lambda x: -x[1][1]):
                print(f"| {100 * us / allus:.2f}% | {n} | {us / n:.1f} | `{k}` |")
            return
        for k, (n, us) in sorted(tot.items(), key=lambda x: -x[1][1]):
            print(f"{us / 1e3:10.3f} ms {n:6d}  {k}")
        return
    for k, v in launch.items():
        print(k, v["name"][:40], v.get("launch__grid_size", ""), float(v.get("gpu__time_duration.sum", 0)) / 1e3)


if __name__ == "__main__":
    main()
