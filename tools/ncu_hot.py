"""Hottest SASS instructions of one kernel in an .ncu-rep (source page): samples, executed count, instruction."""
import csv, subprocess, sys
rep, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
sub = sys.argv[4] if len(sys.argv) > 4 else ""  # pick the first launch whose full name contains this
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + pat],
                     capture_output=True, text=True).stdout.splitlines()
# several launches may match: take the first block
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
iS, iA, iN, iE = hdr.index("Source"), hdr.index("Address"), hdr.index("# Samples"), hdr.index("Instructions Executed")
data = [(int(r[iN] or 0), int(r[iE] or 0), idx, r[iS].strip()) for idx, r in enumerate(rows[1:]) if len(r) > iE]
tot = sum(d[0] for d in data)
print("total samples", tot, "instructions", len(data), "warp-instr executed", sum(d[1] for d in data))
for n, e, idx, s in sorted(data, reverse=True)[:top]:
    print(f"{100.0 * n / max(tot, 1):5.1f}%  exec={e:9d}  #{idx:5d}  {s}")
