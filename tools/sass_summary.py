"""cuobjdump -sass of the Taylor tile kernels: instruction counts per kernel + the full listing of one of them.
python tools/sass_summary.py [full-listing pattern, default 'ILi2ELi5ELb1E' = coded DEFER, rows <= 5]"""
import collections, re, subprocess, sys, os, tempfile
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
csrc = os.path.join(root, "paper_2603_07341_b200", "csrc")
pick = sys.argv[1] if len(sys.argv) > 1 else "ILi2ELi5ELb1ELb0E"
obj = os.path.join(tempfile.gettempdir(), "taylor_sass.o")
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-lineinfo", "-fmad=false",
                       "-c", "-o", obj, "taylor.cu"], cwd=csrc)
sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs, cur, name = collections.OrderedDict(), None, None
for ln in sass.splitlines():
    m = re.search(r"Function : (\S+)", ln)
    if m:
        name = m.group(1)
        cur = funcs.setdefault(name, [])
    if cur is not None:
        cur.append(ln)
print("# cuobjdump -sass of the tile Taylor kernels (taylor.cu, namespace tile), sm_100a")
print("# taylor_tile_kernel<MODE, MAXR, CODED, SHARD>: MODE 0 SINGLE, 1 FIRST, 2 DEFER, 3 CATCHUP; MAXR = row-length bound;")
print("# SHARD 1 = a rank's rows of a sharded space (row filter by halo columns, sums deposited for the all-reduce);")
print("# CODED 1 = 2-byte value codes + shared-memory table.  UBLKCP = cp.async.bulk (bulk copy global -> shared),")
print("# PREEXIT / ACQBULK = griddepcontrol.launch_dependents / griddepcontrol.wait (programmatic dependent launch),")
print("# SYNCS = mbarrier operations, LDG = gathers of x / c / previous term, LDS = slices + value table")
ops = ["UBLKCP", "SYNCS", "PREEXIT", "ACQBULK", "LDG", "LDS", "STG", "DMUL", "DADD", "DFMA", "BAR"]
for fn, lines in funcs.items():
    m = re.search(r"taylor_tile_kernelILi(\d)ELi(\d)ELb([01])ELb([01])E", fn)
    if not m:
        continue
    body = [l for l in lines if re.search(r"/\*[0-9a-f]{4}\*/", l)]
    cnt = {o: sum(1 for l in body if re.search(r"\b" + o + r"\b|\b" + o + r"\.", l)) for o in ops}
    print(f"taylor_tile_kernel<{m.group(1)},{m.group(2)},{m.group(3)},{m.group(4)}>: " + " ".join(f"{o}={cnt[o]}" for o in ops) + f" instructions={len(body)}")
for fn, lines in funcs.items():
    if pick in fn and "taylor_tile_kernel" in fn:
        print("\n# full listing:", fn)
        print("\n".join(lines))
        break
