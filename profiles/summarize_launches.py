"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per kernel name, launch count, mean and total device time (cold-cache,
serialised — compare SHARES, not absolutes)."""
import collections
import csv
import sys


def summarize(path):
    hdr, data = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        name = d["Kernel Name"].split("(")[0].replace("<unnamed>::", "")
        agg.setdefault(name, []).append(float(d["Metric Value"]) / 1e6)
    tot = sum(sum(v) for v in agg.values())
    lines = ["| kernel | launches | mean ms | total ms | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{k}` | {len(v)} | {sum(v)/len(v):.3f} | {sum(v):.2f} | {sum(v)/tot:.1%} |")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summarize(sys.argv[1]))
