"""world_size-2 gloo tests of bench.py's multi-rank host logic (CPU only).

bench.py --gpus N runs one process per GPU; every rank propagates its own N
subintervals (independent fine propagators, no data-path collective, DESIGN.md
§7) from rank-seeded start states, and the timed region is the MAX of the
ranks' device times."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist
    import bench
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # ranks time different amounts; every rank must see the slowest one
    t = bench.max_over_ranks_of(100.0 + 7.0 * rank, world, "cpu")
    np.save(os.path.join(out_dir, f"t{rank}.npy"), np.array([t]))
    dist.barrier()
    dist.destroy_process_group()


def test_max_over_ranks_gloo_world2(tmp_path):
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        assert float(np.load(tmp_path / f"t{r}.npy")[0]) == 107.0


def test_rank_start_states_are_disjoint_seeds():
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench
    import paper_1905_13076_b200 as ps

    class P:
        dim = 37
    a, b = bench.start_states(P, 5, 0), bench.start_states(P, 5, 1)
    assert a.shape == (5, 37) and not np.any(np.all(a == b, axis=1))
    assert np.array_equal(b[2], ps.seeded_normal(bench.SEED + 1 * 5 + 3, 37, 1e-3))
