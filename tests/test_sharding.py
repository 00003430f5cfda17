"""Host-side multi-GPU logic on CPU: world_size-2 gloo processes shard a batch by run id and
gather the records in run-id order; the result equals the single-process batch."""
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2404_18034_b200 import scenario, sharding
from paper_2404_18034_b200.binding import RECORD_DTYPE

ROOT = Path(__file__).resolve().parent.parent


def fake_run_batch(sc, count, first):
    """Records whose fields are pure functions of the run id (what the device produces)."""
    rec = np.zeros(count, RECORD_DTYPE)
    for i in range(count):
        rid = first + i
        init = scenario.disperse(sc, rid)
        rec["run_id"][i] = rid
        rec["initial_position"][i] = init[1:4]
        rec["scp_iterations"][i] = 25
        rec["propellant_used"][i] = (scenario.run_seed(sc.dispersion.seed, rid) % 1000) * 1e-3
    return rec


def test_shard_ranges_partition_the_batch():
    for total in (0, 1, 7, 4096, 65536, 65537):
        for world in (1, 2, 3, 8):
            pos = 0
            sizes = []
            for r in range(world):
                first, count = sharding.shard_range(total, world, r)
                assert first == pos
                pos += count
                sizes.append(count)
            assert pos == total and max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        sharding.shard_range(10, 2, 2)


WORKER = r'''
import sys, numpy as np, torch.distributed as dist
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
from paper_2404_18034_b200 import scenario, sharding
from test_sharding import fake_run_batch
dist.init_process_group("gloo")
sc = scenario.default_scenario(15)
total = int(sys.argv[2])
out = sharding.run_batch_sharded(lambda c, f: fake_run_batch(sc, c, f), total)
t = sharding.max_over_ranks(1.0 + dist.get_rank())
assert t == float(dist.get_world_size())
if dist.get_rank() == 0:
    np.save(sys.argv[3], out)
else:
    assert out is None
dist.destroy_process_group()
'''


@pytest.mark.parametrize("total", [1, 9, 16])  # 1: rank 1 has an empty range
def test_two_rank_gloo_gather_matches_single_process(tmp_path, total):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    out = tmp_path / "records.npy"
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE="2")
    procs = [subprocess.Popen([sys.executable, str(script), str(ROOT), str(total), str(out)],
                              env=dict(env, RANK=str(r), LOCAL_RANK=str(r))) for r in range(2)]
    for p in procs:
        assert p.wait(timeout=180) == 0
    got = np.load(out)
    want = fake_run_batch(scenario.default_scenario(15), total, 0)
    assert got.dtype == want.dtype
    for f in RECORD_DTYPE.names:
        np.testing.assert_array_equal(got[f], want[f])
    np.testing.assert_array_equal(got["run_id"], np.arange(total))
