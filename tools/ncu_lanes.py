"""Per source line of one kernel in an ncu report: warp instructions executed, share, and average active threads
per instruction (divergence map). Usage: python tools/ncu_lanes.py report.ncu-rep [kernel-substring] [top_n]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    ksub = sys.argv[2] if len(sys.argv) > 2 else ""
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fn, hdr, agg, cur = "", None, {}, None
    for r in rows:
        if not r:
            continue
        if r[0] == "Function Name":
            cur = r[1]
            continue
        if r[0] == "File Path":
            fn = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or (ksub and ksub not in (cur or "")):
            continue
        if not r[0].isdigit():
            continue
        try:
            ie = float(r[hdr.index("Instructions Executed")])
            te = float(r[hdr.index("Thread Instructions Executed")])
        except (ValueError, IndexError):
            continue
        if ie <= 0:
            continue
        k = (fn, r[0], r[1][:90])
        a = agg.setdefault(k, [0.0, 0.0])
        a[0] += ie
        a[1] += te
    tot = sum(v[0] for v in agg.values())
    ttot = sum(v[1] for v in agg.values())
    print(f"warp instructions {tot:.4e}, thread instructions {ttot:.4e}, avg active {ttot / max(tot, 1):.2f}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100 * v[0] / tot:6.2f}%  thr/inst {v[1] / v[0]:5.1f}  {k[0]}:{k[1]}  {k[2]}")


if __name__ == "__main__":
    main()


def ranges(rep, ksub, spans):
    """Sum warp/thread instructions per named line span of simulate_lane.cu: spans = [(name, lo, hi), ...]."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, cur, fn = None, None, ""
    acc = {n: [0.0, 0.0] for n, _, _ in spans}
    acc["other"] = [0.0, 0.0]
    for r in rows:
        if not r:
            continue
        if r[0] == "Function Name":
            cur = r[1]
            continue
        if r[0] == "File Path":
            fn = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0].isdigit() or (ksub and ksub not in (cur or "")):
            continue
        try:
            ie = float(r[hdr.index("Instructions Executed")])
            te = float(r[hdr.index("Thread Instructions Executed")])
        except (ValueError, IndexError):
            continue
        ln = int(r[0])
        name = "other"
        if fn == "simulate_lane.cu":
            for n, lo, hi in spans:
                if lo <= ln <= hi:
                    name = n
                    break
        acc[name][0] += ie
        acc[name][1] += te
    tot = sum(v[0] for v in acc.values())
    for n, v in acc.items():
        print(f"{n:10s} {100 * v[0] / tot:6.2f}%  thr/inst {v[1] / max(v[0], 1):5.1f}")
