"""world_size-2 gloo tests of the multi-rank host logic (CPU only)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1905_13076_b200.sharding import shard


def test_shard_covers_everything_once():
    for n in (1, 7, 20, 100, 256):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                first, count = shard(n, r, world)
                seen.extend(range(first, first + count))
            assert seen == list(range(1, n + 1))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_path):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import torch.distributed as dist
    import paper_1905_13076_b200 as ps
    from oracle import pyoracle as po
    from paper_1905_13076_b200.sharding import sharded_fine_phase
    from helpers import NEWTON_BASELINE
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    prob = ps.build_polar_cable(nr=8, ntheta=12)
    mesh = ps.TimeMesh(6, 3, prob.period)
    orc = po.Oracle(prob)
    U = np.stack([ps.seeded_normal(100 + n, prob.dim, 1e-4) for n in range(6)])
    F = sharded_fine_phase(lambda n0, Us: orc.fine_propagate_batch(mesh, n0, Us, newton=NEWTON_BASELINE,
                                                                   mode=po.DIRECT, workers=1), U, rank, world)
    if rank == 0:
        np.save(out_path, F)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_fine_phase_gloo_world2(tmp_path):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(root, "tests"))
    import paper_1905_13076_b200 as ps
    from oracle import pyoracle as po
    from helpers import NEWTON_BASELINE
    out = str(tmp_path / "F.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    F = np.load(out)
    prob = ps.build_polar_cable(nr=8, ntheta=12)
    mesh = ps.TimeMesh(6, 3, prob.period)
    U = np.stack([ps.seeded_normal(100 + n, prob.dim, 1e-4) for n in range(6)])
    ref = po.Oracle(prob).fine_propagate_batch(mesh, 1, U, newton=NEWTON_BASELINE, mode=po.DIRECT, workers=1)
    assert np.array_equal(F, ref)
