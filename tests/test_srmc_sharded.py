"""SRMC sharded solve on CPU (gloo, world_size 2 and 3): north_star item 5.

srmc.solve_sharded partitions the hypercubes over the ranks, runs each backward step on
the rank's own cells and all-gathers the step's y table before the next step (NCCL on
B200s; gloo here). The per-range step is the oracle's (oracle/srmc_oracle.c,
srmc_oracle_step) instead of the CUDA kernel, so this checks the partition, the exchange
and the bitwise G-invariance of the result; the kernel's own per-range entry
(qrmc_srmc_step_device) is covered on the GPU by test_srmc.py."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASES = {
    "sin-lp1": lambda srmc: (srmc.sin_bench_problem(2), srmc.config(4, 7, 40, basis=srmc.LP1, seed=5), True),
    "bergman-lp1": lambda srmc: (srmc.bergman_problem(2, 0.05, 0.2, 0.01, 0.06, 100.0, 0.5),
                                 srmc.config(3, 5, 48, basis=srmc.LP1, lo=4.0, hi=5.2, seed=9), True),
    "sin-lp0": lambda srmc: (srmc.sin_bench_problem(3), srmc.config(3, 4, 33, basis=srmc.LP0, seed=3), False),
}


def _worker(rank, world, port_no, out_dir, case):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "tests"))
    import oracles
    from paper_2407_21084_b200 import srmc
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p, c, with_z = CASES[case](srmc)
    t = srmc.solve_sharded(p, c, with_z=with_z, step_fn=oracles.srmc_oracle_step_fn(p, c))
    np.save(os.path.join(out_dir, f"y{rank}.npy"), t.y)
    if with_z:
        np.save(os.path.join(out_dir, f"z{rank}.npy"), t.z)
    np.save(os.path.join(out_dir, f"r{rank}.npy"), np.array(t.stats["cells"]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", list(CASES))
def test_sharded_srmc_is_bitwise_world_invariant(tmp_path, world, case):
    import oracles
    from paper_2407_21084_b200 import srmc
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), case), nprocs=world, join=True)
    p, c, with_z = CASES[case](srmc)
    y, z = oracles.srmc_port().solve(p, c, with_z=with_z)
    cells = c.cells_per_dim ** p.dim
    ranges = [tuple(np.load(tmp_path / f"r{r}.npy")) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == cells
    assert all(ranges[r][1] == ranges[r + 1][0] for r in range(world - 1))
    for r in range(world):
        assert np.array_equal(np.load(tmp_path / f"y{r}.npy"), y)
        if with_z:
            assert np.array_equal(np.load(tmp_path / f"z{r}.npy"), z)
