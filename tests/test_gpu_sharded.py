"""Sharded (multi-GPU) path on ONE GPU: WORLD_SIZE ranks share cuda:0 and exchange through gloo (host-staged
callbacks), so the full key-hash sharding logic -- candidate routing, look-up requests, halo exchange, distributed
radix select, tie draw -- runs on the real kernels and is compared with the oracle bit for bit.  The NCCL transport
differs only inside paper_2603_07341_b200/dist.py."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _launch(world, names, steps, port):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "tests", "dist_worker.py"), names, str(steps)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-6000:])
    assert "SHARDED_OK" in r.stdout, r.stdout[-3000:]
    return r.stdout


@pytest.mark.gpu
def test_two_ranks_match_oracle():
    _launch(2, "cfg1_holstein_L4_d8,ties_holstein_L5_d6,cube_2x2x2_d16,disordered_4x3_d7", 30, 29611)


@pytest.mark.gpu
def test_three_and_four_ranks_match_oracle():
    _launch(3, "ties_holstein_L5_d6,square_3x3_d5", 25, 29612)
    _launch(4, "cfg2_layout_L16_d16_small,substeps_L4_d4_m1,tb_chain_31", 20, 29613)
