"""Transport over peer memory (hk_transport_rhs_peer + CUDA IPC, PartitionPeerHalo).

Two processes, each one x-slab rank, both on cuda:0 (this box has one GPU):
their kernels never wait on each other — a host barrier orders the slab
writes before the reads — so the IPC mapping and the ghost-column addressing
are exercised exactly as across NVLink, without standing in for a second
GPU's timing.  World 1 maps its own slab (periodic wrap)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("world", [1, 2, 3])
def test_peer_transport_matches_global(world):
    env = dict(os.environ, WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(29620 + world))
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "peer_worker.py")], env=dict(env, RANK=str(r)),
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for r in range(world)]
    outs = [p.communicate(timeout=300)[0] for p in procs]
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o
