"""Per-basic-block view of an ncu SASS source page (ncu -i rep --page source --csv --print-source=sass):
consecutive instructions executed the same number of times form one block; prints each block's share of the
kernel's warp instructions, its active lanes per instruction, and its first/last SASS lines.
Usage: python tools/ncu_sass.py page.csv [min_share_pct]"""
import csv
import sys


def main():
    path = sys.argv[1]
    thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    ia, isrc, iex, ith = (hdr.index(k) for k in ("Address", "Source", "Instructions Executed",
                                                  "Thread Instructions Executed"))
    ins = []
    for r in rows[hdr_i + 1:]:
        if len(r) <= ith or not r[ia].startswith("0x"):
            continue
        ins.append((int(r[ia], 16), r[isrc].strip(), int(float(r[iex] or 0)), int(float(r[ith] or 0))))
    base = ins[0][0]
    total = sum(x[2] for x in ins)
    tthr = sum(x[3] for x in ins)
    print(f"warp instructions {total:.4e}, thread instructions {tthr:.4e}, lanes/instr {tthr / max(total, 1):.2f}")
    blocks = []
    cur = []
    for x in ins:
        if cur and x[2] != cur[-1][2]:
            blocks.append(cur)
            cur = []
        cur.append(x)
    if cur:
        blocks.append(cur)
    for b in blocks:
        ex = sum(x[2] for x in b)
        th = sum(x[3] for x in b)
        if ex / total * 100 < thr:
            continue
        print(f"{ex / total * 100:6.2f}%  n={len(b):3d} x{b[0][2]:>11d} lanes={th / max(ex, 1):5.1f}  "
              f"{b[0][0] - base:05x}-{b[-1][0] - base:05x}  {b[0][1][:60]} ... {b[-1][1][:50]}")


if __name__ == "__main__":
    main()
