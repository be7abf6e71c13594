"""Per-source-line stall samples / executed instructions of one kernel in an .ncu-rep captured with
`ncu --set full --import-source on` from a -lineinfo build:  python tools/ncu_lines.py REP KERNEL_REGEX [TOP] [0=by samples|1=by instructions]"""
import collections, csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur, agg = None, collections.OrderedDict()
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur = r[1].split("/")[-1]
    elif r[0] == "Line No":
        iS = r.index("Warp Stall Sampling (All Samples)"); iI = r.index("Instructions Executed")
    elif r[0] != "Function Name" and len(r) > 3 and r[2] == "-":
        try:
            k = (cur, int(r[0]), r[1].strip()[:90]); a = agg.get(k, (0, 0)); agg[k] = (a[0] + int(r[iS]), a[1] + int(r[iI]))
        except Exception: pass
tS = sum(v[0] for v in agg.values()) or 1; tI = sum(v[1] for v in agg.values()) or 1
print(f"samples {tS}  warp-instructions {tI}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][int(sys.argv[4]) if len(sys.argv) > 4 else 0])[:top]:
    print(f"{k[0]:12s}{k[1]:5d} samp={100 * v[0] / tS:5.1f}% instr={100 * v[1] / tI:5.1f}%  {k[2]}")
