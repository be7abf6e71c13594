"""Instruction mix of one kernel in an .ncu-rep (source page): warp-level executed counts by opcode."""
import csv, subprocess, sys, collections
rep, pat = sys.argv[1], sys.argv[2]
sub = sys.argv[3] if len(sys.argv) > 3 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + pat],
                     capture_output=True, text=True).stdout.splitlines()
blocks, cur = [], None
for ln in out:
    if ln.startswith('"Kernel Name"'):
        cur = []
        if sub in ln:
            blocks.append(cur)
    elif cur is not None:
        cur.append(ln)
rows = list(csv.reader(blocks[0]))
hdr = rows[0]
iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
mix = collections.Counter()
tot = 0
for r in rows[1:]:
    if len(r) <= iE:
        continue
    e = int(r[iE] or 0)
    toks = r[iS].strip().split()
    op = toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?")
    mix[op.split(".")[0]] += e
    tot += e
print("warp instructions executed:", tot)
for op, e in mix.most_common(30):
    print(f"{100.0 * e / tot:5.1f}%  {e:10d}  {op}")
