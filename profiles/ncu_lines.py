"""Per-source-line hot spots of one kernel in an ncu report (warp-stall samples,
instructions executed, L2 sectors), from `ncu --page source --print-source cuda,sass`.

    python profiles/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [top]
"""
import csv
import io
import subprocess
import sys


def main(rep, kregex, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kregex,
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    agg, fname, hdr = {}, "?", None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = {h: i for i, h in enumerate(r)}
            continue
        if hdr is None or r[0] in ("", "Function Name"):
            continue
        try:
            line = int(r[0])
        except ValueError:
            continue
        def num(col):
            i = hdr.get(col)
            try:
                return float(r[i]) if i is not None else 0.0
            except ValueError:
                return 0.0
        key = (fname, line, r[1][:70])
        a = agg.setdefault(key, [0.0, 0.0, 0.0])
        a[0] += num("Warp Stall Sampling (All Samples)")
        a[1] += num("Instructions Executed")
        a[2] += num("L2 Theoretical Sectors Global")
    tot = [sum(v[i] for v in agg.values()) or 1 for i in range(3)]
    print(f"{'file:line':32s} {'stall%':>7s} {'inst%':>7s} {'L2sec%':>7s}  source")
    for (f, l, s), v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(top)]:
        print(f"{f + ':' + str(l):32s} {100 * v[0] / tot[0]:7.2f} {100 * v[1] / tot[1]:7.2f} "
              f"{100 * v[2] / tot[2]:7.2f}  {s}")


if __name__ == "__main__":
    main(*sys.argv[1:])
