"""Multi-GPU host logic on CPU: 2 ranks over gloo (127.0.0.1).

Each rank plays one GPU's GVM. It folds its SPMD workers' NAS EP partials
(class S split over 4 workers, two per rank) into a per-GPU record. The
records are all-gathered (gloo here, NCCL via vgpu_cu_reduce_final on B200)
and every rank folds them in rank order. Checks: all ranks hold bit-identical
results, the counts equal the single-process oracle exactly, and the sums
pass NPB's verification (1e-8).
"""
import os
import struct
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle
from paper_1511_07658_b200 import reduce as R


def _worker_result(worker, part):
    b = lambda x: struct.pack("<d", x)[::-1].hex()  # big-endian hex of the LE bits
    return {"worker": worker, "checksum": "1",
            "ep": {"sx_bits": b(part.sx), "sy_bits": b(part.sy), "pairs": part.pairs,
                   "n_batches": part.n_batches, "q": list(part.q)}}


def _rank_main(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    workers = [2 * rank, 2 * rank + 1]
    results = [_worker_result(w, oracle.ep_job(24, 64 * w, 64)) for w in workers]
    rec = torch.tensor(R.record_from_workers(results), dtype=torch.float64)
    gathered = [torch.zeros_like(rec) for _ in range(world)]
    dist.all_gather(gathered, rec)
    flat = torch.cat(gathered).tolist()
    folded = R.fold_in_rank_order(flat, world)
    out_q.put((rank, folded))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bits_helper_roundtrip():
    x = -3247.834652034623
    h = struct.pack("<d", x)[::-1].hex()
    assert R.bits_to_double(h) == x


def test_two_rank_final_reduce_is_deterministic_and_exact():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a, b = got[0], got[1]
    assert struct.pack("<16d", *a) == struct.pack("<16d", *b)  # identical on every rank
    whole = oracle.ep_job(24, 0, 256)
    assert [int(x) for x in a[1:11]] == list(whole.q)
    assert int(a[13]) == whole.pairs == 13176389
    v = R.ep_verdict(a, 24)
    assert v["verified"], v
    assert a[0] == 4.0  # jobs folded
