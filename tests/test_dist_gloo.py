"""Multi-rank path on CPU (gloo, world_size 2): structure sharding and the
row-order gather reproduce the single-process batch bit for bit. The per-rank
solve here is the oracle (no GPU in this container); bench.py runs the same
sharding with the device path under torchrun."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    sys.path.insert(0, os.path.join(ROOT, "oracle", "_build"))
    import torch.distributed as dist

    import harness as H
    import mb_oracle
    from paper_2306_00271_b200 import configs
    from paper_2306_00271_b200.dist import gather_rows, shard_pairs
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = configs.config2(n_structures=5).subset(theta0=[0.7, 3.1], slices=40)
    pairs = [(s, t0, t1) for s in range(len(w.structures)) for t1 in w.theta1 for t0 in w.theta0]
    lo, hi, idx, local = shard_pairs(pairs, len(w.structures), rank, world)
    part = w.subset(structures=list(range(lo, hi)))
    eta, _, _ = H.run_oracle(mb_oracle, part, threads=1) if hi > lo else (np.zeros((0, w.n_rods)), None, None)
    full = gather_rows(eta, idx, len(pairs))
    if rank == 0:
        np.save(os.path.join(outdir, "gathered.npy"), full)
    dist.barrier()
    dist.destroy_process_group()


def test_shard_boundaries():
    from paper_2306_00271_b200.dist import shard_structures
    for S in (1, 5, 1024):
        for world in (1, 2, 3, 8):
            blocks = [shard_structures(S, r, world) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == S
            assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))
            assert max(b[1] - b[0] for b in blocks) - min(b[1] - b[0] for b in blocks) <= 1


def test_two_rank_gather_matches_single(oracle, tmp_path):
    import harness as H
    from paper_2306_00271_b200 import configs
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True, start_method="spawn")
    w = configs.config2(n_structures=5).subset(theta0=[0.7, 3.1], slices=40)
    ref, _, _ = H.run_oracle(oracle, w, threads=1)
    assert np.array_equal(np.load(tmp_path / "gathered.npy"), ref)
