"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per kernel launch count, mean duration (us) and share of the total."""
import collections
import csv
import sys


def summarise(path, top=20):
    hdr = None
    agg = collections.defaultdict(list)
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(d.get("Metric Unit", "nsecond"), 1e-3)
                agg[d["Kernel Name"].split("(")[0][:70]].append(float(d["Metric Value"].replace(",", "")) * scale)
    tot = sum(sum(v) for v in agg.values())
    lines = [f"{'kernel':70s} {'n':>5s} {'mean_us':>10s} {'share':>6s}"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1]))[:top]:
        lines.append(f"{k:70s} {len(v):5d} {sum(v)/len(v):10.1f} {100*sum(v)/tot:5.1f}%")
    lines.append(f"total {tot/1e3:.2f} ms over {sum(len(v) for v in agg.values())} launches")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summarise(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20))
