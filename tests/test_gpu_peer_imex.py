"""The x-slab penalized PR(2,2,2) step across 2 and 3 processes (one x-slab
rank each) with the transport reading the neighbours' stage field over CUDA
IPC (partition.PeerHalo, hk_transport_rhs_peer): every rank's slab equals the
world-1 step of the global field bitwise.  The processes share this box's one
GPU; their kernels never wait on each other (host barriers order the stage
writes before the neighbours' reads), so this exercises the IPC mapping, the
ghost-column addressing and the stage ordering exactly as across NVLink."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("world", [1, 2, 3])
def test_peer_imex_step_matches_world1(world):
    env = dict(os.environ, WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(29640 + world))
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "peer_imex_worker.py")], env=dict(env, RANK=str(r)),
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for r in range(world)]
    outs = [p.communicate(timeout=600)[0] for p in procs]
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o
