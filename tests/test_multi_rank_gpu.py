"""The multi-rank path with the CUDA library on every rank: 2 and 3 ranks (gloo, one shared GPU)
each simulate a strong-scaling shard with libmig; the reduced per-policy totals equal one call over all traces, bit
for bit (tools/multi_rank_check.py). CPU-only coverage of the reduce itself is in test_multi_gloo.py."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,cfg", [(2, 3), (3, 5)])
def test_sharded_libmig_totals_equal_single_call(world, cfg):
    port = 29600 + world + cfg
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(ROOT, "tools", "multi_rank_check.py"), "--config", str(cfg), "--traces", "30001"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    assert f"MULTI_RANK_OK {world}" in r.stdout
