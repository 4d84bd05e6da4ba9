"""N > 1 plumbing on CPU: world_size-2 gloo ranks, replica realisations and the
max-over-ranks timing reduction bench.py uses."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp

from paper_1409_2556_b200 import inputs
from paper_1409_2556_b200.replicas import replica_config


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch.distributed as dist

    from paper_1409_2556_b200.replicas import barrier, max_over_ranks
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = replica_config(inputs.config(0).scaled((16, 16)), rank)
    lk, _ = cfg.fields()
    barrier()
    vals = max_over_ranks([10.0 * (rank + 1), -float(rank)])
    out[rank] = (float(lk.sum()), vals)
    dist.destroy_process_group()


def test_two_rank_gloo_replicas_and_max():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert out[0][1] == [20.0, 0.0] and out[1][1] == [20.0, 0.0]
    assert out[0][0] != out[1][0]  # distinct realisations per rank


def test_rank0_replica_is_the_baseline_input():
    cfg = inputs.config(4)
    assert replica_config(cfg, 0).log_kappa == cfg.log_kappa
    r1 = replica_config(cfg, 1)
    assert r1.log_kappa["seed"] != cfg.log_kappa["seed"]
    assert r1.log_storativity["seed"] != cfg.log_storativity["seed"]
    assert np.isclose(r1.log_kappa["var"], cfg.log_kappa["var"])
