"""Per-source-line stall samples / instructions of one kernel from an .ncu-rep (ncu --import-source on, -lineinfo)."""
import collections, csv, subprocess, sys

def main(rep, top=30, key="samp"):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur, agg = None, collections.OrderedDict()
    iS = iI = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
        elif r[0] == "Line No":
            iS = r.index("Warp Stall Sampling (All Samples)")
            iI = r.index("Instructions Executed")
        elif r[0] not in ("Function Name",) and len(r) > 3 and r[2] == "-":
            try:
                agg[(cur, int(r[0]), r[1].strip()[:90])] = (int(r[iS]), int(r[iI]))
            except Exception:
                pass
    tS = sum(v[0] for v in agg.values()) or 1
    tI = sum(v[1] for v in agg.values()) or 1
    print(f"samples {tS}  warp-instructions {tI}")
    idx = 0 if key == "samp" else 1
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][idx])[:top]:
        print(f"{k[0]:12s}{k[1]:5d} samp={100 * v[0] / tS:5.1f}% instr={100 * v[1] / tI:5.1f}%  {k[2]}")

if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30, sys.argv[3] if len(sys.argv) > 3 else "samp")
