"""CPU, world_size 2 over gloo: sharding J draws across ranks by global draw
index reproduces the single-process draw sequence exactly (the property the
multi-GPU bench relies on). Each rank draws with the CPU oracle (the same
CounterRng stream mapping the device kernels use, checked on GPU by
test_gpu_parity.py::test_draw_offset_sharding_matches_one_call)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2301_12584_b200.sharding import sample_sharded, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_range_partitions():
    for J in (1, 2, 7, 8, 65536, 65537):
        for world in (1, 2, 3, 8):
            covered = []
            for r in range(world):
                s, c = shard_range(J, r, world)
                covered.extend(range(s, s + c))
            assert covered == list(range(J))


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from parity_util import config1_factors
    fs = config1_factors(shapes=((500, 8), (300, 8), (257, 8)))
    o = oracle.OracleKrp(fs, "port")

    def fn(excluded, count, seed, offset):
        return o.sample(excluded, count, seed, draw_offset=offset)

    for e in (None, 1):
        idx, prob, rows = sample_sharded(fn, e, 1001, 77, rank, world)
        if rank == 0:
            np.savez(out + f"_{e}.npz", idx=idx, prob=prob, rows=rows)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo_sharding_equals_single_call(tmp_path):
    out = str(tmp_path / "shard")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    import oracle
    from parity_util import config1_factors
    fs = config1_factors(shapes=((500, 8), (300, 8), (257, 8)))
    o = oracle.OracleKrp(fs, "port")
    for e in (None, 1):
        idx, prob, rows = o.sample(e, 1001, 77)
        got = np.load(out + f"_{e}.npz")
        assert np.array_equal(got["idx"], idx)
        assert np.array_equal(got["prob"], prob)
        assert np.array_equal(got["rows"], rows)
