"""Multi-rank host path on CPU (gloo, world_size 2 and 3).

The B200 solve shards paths by the reference's lanes (parallel.hpp:20-36):
rank g owns lanes [g*ceil(256/G), ...), computes their per-lane projection
partials, and one all-gather per backward step gives every rank all 256
lane partials, which each rank sums in lane order 0..255
(solver.cpp:202-209) -- so alpha_i is bitwise independent of G. Here the
per-lane partials come from the CPU oracle and the collective is gloo; the
ownership map is the C library's own (qrmc_gpu_lane_ownership)."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port_no, out_dir):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "tests"))
    import oracles
    from paper_2407_21084_b200 import _abi
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    L = _abi.lib()
    prob = _abi.sin_bench_problem(2)
    paths = 300_000  # 293 chunks: lanes 0..36 hold two chunks, the rest one
    cfg = _abi.ConfigHolder(steps=3, paths=paths, damping=2.1, seed=77, gamma_kind=2, degrees=[4])
    k = oracles.port().gamma(2, 2, [4])[0].shape[0]
    lo, hi, n = C.c_int32(), C.c_int32(), C.c_int64()
    assert L.qrmc_gpu_lane_ownership(paths, rank, world, C.byref(lo), C.byref(hi), C.byref(n)) == 0
    lpr = (256 + world - 1) // world
    _, part = oracles.port().backward_solve_lanes(prob, cfg, k, lo.value, hi.value)
    mine = torch.zeros(lpr, k, dtype=torch.float64)
    mine[: hi.value - lo.value] = torch.from_numpy(part)
    gathered = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(gathered, mine)
    rows = torch.cat(gathered)[:256].numpy()
    coeff0 = np.zeros(k)
    for lane in range(256):  # fixed lane order, exactly the reference's final reduction
        coeff0 = coeff0 + rows[lane]
    coeff0 = coeff0 * (1.0 / paths)
    np.save(os.path.join(out_dir, f"rank{rank}.npy"), coeff0)
    counts = torch.tensor([n.value], dtype=torch.int64)
    dist.all_reduce(counts)
    np.save(os.path.join(out_dir, f"count{rank}.npy"), counts.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_exchange_is_bitwise_world_invariant(tmp_path, port, world):
    from paper_2407_21084_b200 import _abi
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    prob = _abi.sin_bench_problem(2)
    cfg = _abi.ConfigHolder(steps=3, paths=300_000, damping=2.1, seed=77, gamma_kind=2, degrees=[4])
    k = port.gamma(2, 2, [4])[0].shape[0]
    single, _ = port.backward_solve(prob, cfg, k)
    for r in range(world):
        np.testing.assert_array_equal(np.load(tmp_path / f"rank{r}.npy"), single[0])
        assert int(np.load(tmp_path / f"count{r}.npy")[0]) == 300_000
