"""Summarise an ncu report's SASS source page: top stall reasons and hottest instructions.

  python tools/ncu_stalls.py gpurun_out/prof.ncu-rep [n_top]
"""
import csv
import io
import subprocess
import sys


def main(rep, n_top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    data = rows[2:]
    i_s = h.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
    tot = sum(float(r[i_s] or 0) for r in data)
    print(rows[0][0][:160])
    print("total samples", tot)
    agg = {}
    for r in data:
        for i in stall_cols:
            try:
                agg[h[i]] = agg.get(h[i], 0) + float(r[i] or 0)
            except ValueError:
                pass
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:10]:
        print(f"  {k:28s} {100 * v / tot:5.1f}%")
    for r in sorted(data, key=lambda r: -float(r[i_s] or 0))[:n_top]:
        print(f"  {r[0][-5:]} {r[1][:72]:72s} {100 * float(r[i_s]) / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
