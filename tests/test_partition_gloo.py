"""Row-partitioned tree construction, host side on CPU:

* the partition plan (row ranges, per-level compact slot ranges) covers every
  stored node of the reference topology (init_tree, segment_tree_sampler.cpp:111-149)
  exactly once, and each subtree's rows are the rows under its level-g node;
* world_size 2 over gloo: the per-level all-gather of owned slots and the
  subtree-root gather reassemble the oracle's tree, and the top levels reduced
  from the gathered subtree roots equal the oracle's nodes.
The device side (krpg_build_partition / krpg_finish_partitions, bit-identical to
the single build) is covered by test_gpu_parity.py::test_partitioned_build_*."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2301_12584_b200 import _lib
from paper_2301_12584_b200.sharding import exchange_partitioned_tree, partition_slots, tree_geometry

SHAPES = [(4096, 16), (1000, 8), (777, 24), (513, 32), (3000, 40), (2049, 56), (130, 5), (64, 4)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _node_rows(I, F, v):
    f, l, L, n = (C.c_uint64() for _ in range(4))
    _lib.check(_lib.lib().krpg_topology_node_rows(I, F, v, C.byref(f), C.byref(l), C.byref(L), C.byref(n)))
    return f.value, l.value


def _part_rows(I, R, parts, part):
    f, l = C.c_uint64(), C.c_uint64()
    _lib.check(_lib.lib().krpg_partition_rows(I, R, parts, part, C.byref(f), C.byref(l)))
    return f.value, l.value


@pytest.mark.parametrize("I,R", SHAPES)
def test_partition_plan_covers_every_stored_node_once(I, R):
    geo = tree_geometry(I, R)
    L, npos = geo["L"], geo["npos"]
    parts = 2
    while parts <= min(npos, 16):
        g = parts.bit_length() - 1
        owner = np.full(L, -1)
        rows = []
        for part in range(parts):
            # subtree rows = rows of the level-g node (2^g - 1 + part)
            assert _part_rows(I, R, parts, part) == _node_rows(I, R, (1 << g) - 1 + part)
            rows.append(_part_rows(I, R, parts, part))
            for lev, s0, span, valid in partition_slots(I, R, parts, part):
                for s in range(s0 + part * span, s0 + part * span + valid):
                    assert owner[s] == -1
                    owner[s] = part
                    v = 2 * s - 1  # stored heap node of slot s
                    assert (1 << lev) - 1 <= v < (1 << (lev + 1)) - 1  # on tree level lev
                    f, l = _node_rows(I, R, v)
                    assert rows[-1][0] <= f and l <= rows[-1][1]  # inside the subtree
        assert rows[0][0] == 0 and rows[-1][1] == I
        assert all(rows[i][1] == rows[i + 1][0] for i in range(parts - 1))
        # the rest: slots of levels <= g (root, top levels and the stored subtree roots)
        rest = [s for s in range(L) if owner[s] == -1]
        assert rest == list(range(min(L, 1 << g)))
        parts *= 2


def _exchange_worker(rank, world, port, out, I, R):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from parity_util import pareto_factors
    U = pareto_factors([(I, R)], seed=I)[0]
    t = oracle.OracleTree(U, R, None, "port")
    P = R * (R + 1) // 2
    L = tree_geometry(I, R)["L"]
    iu = np.triu_indices(R)
    packed = lambda v: t.node_gram(v)[iu]  # noqa: E731
    tree = torch.full((L * P,), float("nan"), dtype=torch.float64)
    for lev, s0, span, valid in partition_slots(I, R, world, rank):
        for s in range(s0 + rank * span, s0 + rank * span + valid):
            tree[s * P:(s + 1) * P] = torch.from_numpy(packed(2 * s - 1))
    g = world.bit_length() - 1
    subroot = torch.from_numpy(packed((1 << g) - 1 + rank).copy())
    roots = exchange_partitioned_tree(tree, subroot, I, R)
    if rank == 0:
        np.savez(out, tree=tree.numpy(), roots=roots.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("I,R", [(4096, 16), (777, 24)])
def test_two_rank_gloo_tree_exchange(tmp_path, I, R):
    out = str(tmp_path / "tree.npz")
    mp.spawn(_exchange_worker, args=(2, _free_port(), out, I, R), nprocs=2, join=True)
    import oracle
    from parity_util import pareto_factors
    U = pareto_factors([(I, R)], seed=I)[0]
    t = oracle.OracleTree(U, R, None, "port")
    P = R * (R + 1) // 2
    L = tree_geometry(I, R)["L"]
    iu = np.triu_indices(R)
    got = np.load(out)
    tree, roots = got["tree"].reshape(L, P), got["roots"].reshape(2, P)
    for s in range(1, L):  # every slot below level 1 came through the exchange
        if s == 1:
            continue  # level-1 left child = subtree root 0, written by finish from `roots`
        assert np.array_equal(tree[s], t.node_gram(2 * s - 1)[iu]), s
    assert np.array_equal(roots[0], t.node_gram(1)[iu]) and np.array_equal(roots[1], t.node_gram(2)[iu])
    # the top level from the gathered roots (parent = left + right, :185)
    assert np.array_equal(roots[0] + roots[1], t.node_gram(0)[iu])
