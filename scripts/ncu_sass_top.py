"""Top SASS instructions of an ncu --set full report by warp-stall samples (and executed count).

usage: python scripts/ncu_sass_top.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30
    r = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                       capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(r.stdout)))
    i0 = next(i for i, x in enumerate(rows) if x and x[0] == "Address")
    h = rows[i0]
    ix = {k: i for i, k in enumerate(h)}
    data = [x for x in rows[i0 + 1:] if len(x) == len(h)]
    S, E = ix["Warp Stall Sampling (All Samples)"], ix["Instructions Executed"]
    f = lambda v: float(v) if v not in ("", "-") else 0.0
    tot_s, tot_e = sum(f(x[S]) for x in data), sum(f(x[E]) for x in data)
    print(f"samples {tot_s:.0f}  warp instructions {tot_e:.0f}")
    ops = {}
    for x in data:
        op = x[ix["Source"]].split()[0] if x[ix["Source"]].split() else "?"
        if op.startswith("@"):
            op = x[ix["Source"]].split()[1]
        op = op.split(".")[0]
        a = ops.setdefault(op, [0.0, 0.0])
        a[0] += f(x[S]); a[1] += f(x[E])
    print("by opcode (stall %, instr %):", ", ".join(f"{k} {v[0]/tot_s*100:.1f}/{v[1]/tot_e*100:.1f}"
                                              for k, v in sorted(ops.items(), key=lambda kv: -kv[1][0])[:16]))
    for j, x in sorted(enumerate(data), key=lambda jx: -f(jx[1][S]))[:top]:
        print(f"{j:5d} {f(x[S])/tot_s*100:5.1f}% {f(x[E])/tot_e*100:5.1f}%  {x[ix['Source']][:90]}")


if __name__ == "__main__":
    main()
