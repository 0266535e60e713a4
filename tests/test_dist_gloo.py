"""Multi-rank path on CPU (gloo, world_size 2): frames shard by global id with no data-path
exchange and the counters meet in one SUM all-reduce.  The per-rank decode
here is the oracle (test infrastructure), so the test checks the sharding and the collective,
not the kernels: the reduced counters must equal a single-process run over all frames."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
import oracle
import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _counters(name, a, b):
    w = synth.workload(name)
    oc = oracle.Code(w.shifts(), w.Z)
    x, y, _ = w.gen(a, b - a)
    syn = oc.syndrome(x)
    r = oc.decode(oc.build_llr(w.qber, y), syn, w.max_iter, 1, want_state=False, nthreads=2)
    err = np.unpackbits(r["bits"] ^ x, axis=1, bitorder="little")[:, : w.n].sum(1)
    return np.array([b - a, r["success"].sum(), (err > 0).sum(), ((err > 0) & (r["success"] == 1)).sum(),
                     r["iters"].sum()], dtype=np.int64)


def _worker(rank, world, port, name, F, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, b = bench.shard(F, rank, world)
    c = torch.from_numpy(_counters(name, a, b))
    bench.reduce_counters(c, world)
    if rank == 0:
        out.put(c.numpy().tolist())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("F", [48, 37])
def test_two_rank_counters_equal_single_process(F):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, "C2", F, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = q.get(timeout=300)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == _counters("C2", 0, F).tolist()


def test_shards_cover_every_frame_once():
    for F in (1, 7, 65536, 65537):
        for world in (1, 2, 3, 4, 8):
            ids = np.concatenate([np.arange(*bench.shard(F, r, world)) for r in range(world)])
            assert np.array_equal(ids, np.arange(F))
