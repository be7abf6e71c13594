"""Registers / spills of the Taylor tile kernels from an `nvcc -Xptxas -v` log."""
import re, sys
t = open(sys.argv[1]).read()
for m in re.finditer(r"Compiling entry function '([^']+)'[^\n]*\n[^\n]*\n\s*(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads\n[^\n]*Used (\d+) registers", t):
    mm = re.search(r"taylor_tile_kernelILi(\d)ELi(\d)EL[bi]([012])", m.group(1))
    if mm:
        print("mode", mm.group(1), "maxr", mm.group(2), "coded", mm.group(3), "stack", m.group(2), "spill", m.group(3), "regs", m.group(5))
