"""Top stalled SASS instructions of an `ncu --page source --csv --print-source cuda,sass` export,
with the nearest preceding CUDA source line and the stall reasons of each:

    python tools/ncu_stalls.py SRC.csv[.gz] [--top 30]
"""
import csv
import gzip
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30
    rows = list(csv.reader((gzip.open if path.endswith(".gz") else open)(path, "rt")))
    insts, src, total = [], "", 0
    head = None
    for r in rows:
        if r and r[0] == "Line No":
            head = r
            continue
        if head is None or len(r) < len(head):
            continue
        if r[2] == "-" or not r[2].startswith("0x"):  # a source line
            src = f"{r[0]}: {r[1].strip()[:70]}"
            continue
        samples = int(r[4]) if r[4].isdigit() else 0
        total += samples
        reasons = {head[i][6:]: int(r[i]) for i in range(len(head))
                   if head[i].startswith("stall_") and "Not Issued" not in head[i] and r[i].isdigit() and r[i] != "0"}
        insts.append((samples, r[3].strip()[:60], src, reasons))
    insts.sort(key=lambda t: -t[0])
    print(f"total samples {total}")
    for s, sass, line, reasons in insts[:top]:
        rs = ", ".join(f"{k} {v}" for k, v in sorted(reasons.items(), key=lambda kv: -kv[1])[:3])
        print(f"{s:7d} {100 * s / total:5.1f}%  {sass:<60} | {line} | {rs}")


if __name__ == "__main__":
    main()
