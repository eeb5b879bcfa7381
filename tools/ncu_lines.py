"""Aggregate an ncu source page (--page source --csv --print-source cuda,sass)
per CUDA source line: warp instructions executed and stall samples.

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_lines.py src.csv [top]
"""
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    rows, fname, hdr = [], None, None
    with open(path) as f:
        for r in csv.reader(f):
            if not r:
                continue
            if r[0] == "File Path":
                fname = r[1].split("/")[-1]
                continue
            if r[0] == "Line No":
                hdr = r
                continue
            if hdr is None or not r[0].isdigit() or r[2] != "-":
                continue
            d = dict(zip(hdr[2:], r[2:]))
            rows.append((fname, int(r[0]), r[1].strip()[:70], int(d.get("Instructions Executed", 0) or 0),
                         int(d.get("Warp Stall Sampling (All Samples)", 0) or 0)))
    ti = sum(x[3] for x in rows) or 1
    ts = sum(x[4] for x in rows) or 1
    print(f"total warp instructions {ti:.3e}, samples {ts}")
    for fn, ln, src, ins, smp in sorted(rows, key=lambda x: -x[3])[:top]:
        print(f"{100 * ins / ti:5.1f}% inst {100 * smp / ts:5.1f}% smp  {fn}:{ln}  {src}")


if __name__ == "__main__":
    main()
