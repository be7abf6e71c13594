"""Does PCIe DMA traffic slow the resident step?  Resident C2 steps alone, beside back-to-back H2D copies, beside D2H
copies and beside both (pinned 40 MB buffers on a side stream): the Taylor phase's time per step in each case."""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_07341_b200 as pb

model = dict(kind=1, extents=(16,), eps=(0.0,), hop=(1.0,), omega=(1.0,), g=(1.0,), d_pho=16)
ctx = pb.Context(pb.ModelDef(**model))
run = ctx.run(init="localized", site=-1, m_init=10, m=2, q_nom=1000000, dt=0.05, rtol=1e-15, t_max=50.0, seed=7)
for _ in range(12):
    run.step()
nbytes = 40 << 20
h_up = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
h_dn = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
d_up = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
d_dn = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
s_up, s_dn = torch.cuda.Stream(), torch.cuda.Stream()
stop = False


def pump(up, dn):
    while not stop:
        if up:
            with torch.cuda.stream(s_up):
                for _ in range(4):
                    d_up.copy_(h_up, non_blocking=True)
        if dn:
            with torch.cuda.stream(s_dn):
                for _ in range(4):
                    h_dn.copy_(d_dn, non_blocking=True)
        s_up.synchronize()
        s_dn.synchronize()


for name, up, dn in (("alone", False, False), ("beside H2D", True, False), ("beside D2H", False, True), ("beside both", True, True)):
    stop = False
    th = None
    if up or dn:
        th = threading.Thread(target=pump, args=(up, dn))
        th.start()
        time.sleep(0.05)
    run.reset_times()
    for _ in range(20):
        run.step()
    tm = run.times()
    stop = True
    if th:
        th.join()
    print(f"{name:12s}: step {tm['total_ms']:.3f} ms (select {tm['select_ms']:.3f} adapt {tm['grow_ms']:.3f} expmv {tm['expmv_ms']:.3f})", flush=True)
