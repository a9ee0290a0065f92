"""Aggregate an ncu source page (--page source --csv --print-source=cuda,sass) per CUDA source line:
instructions executed and stall samples. Usage: python tools/ncu_lines.py report.ncu-rep [top_n]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    agg = {}
    fname = "?"
    hdr = None
    cur = None
    total = 0
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8:
            continue
        if r[0]:
            cur = (fname, int(r[0]), r[1].strip()[:90])
        if r[2]:
            try:
                n = int(float(r[hdr.index("Instructions Executed")]))
                s = int(float(r[hdr.index("Warp Stall Sampling (All Samples)")]))
            except (ValueError, IndexError):
                continue
            a = agg.setdefault(cur, [0, 0])
            a[0] += n
            a[1] += s
            total += n
    print(f"total warp instructions executed: {total:.4e}")
    for k, (n, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{n / total * 100:6.2f}%  stall_samples={s:7d}  {k[0]}:{k[1]}  {k[2]}")


if __name__ == "__main__":
    main()
