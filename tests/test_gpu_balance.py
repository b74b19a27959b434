"""Dynamic load balancing of the layer-2 residuals (SURVEY §8f "next" #3)
wired into the x-slab hybrid step through hk_hybrid_step's residual hook:
with 2 and 3 x-slab ranks (processes sharing this box's GPU, the exchange
staged through host memory on gloo) the balanced step equals the unbalanced
step bitwise and cells actually move between ranks."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("world", [1, 2, 3])
def test_balanced_hybrid_step_is_bitwise(world):
    env = dict(os.environ, WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(29660 + world))
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "balance_worker.py")], env=dict(env, RANK=str(r)),
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for r in range(world)]
    outs = [p.communicate(timeout=600)[0] for p in procs]
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o
