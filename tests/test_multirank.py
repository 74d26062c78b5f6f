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


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_weak_scaling_ep_slices(world):
    """bench.py's N-GPU EP problem: every GPU keeps 4096 batches (one class A)
    split over its 8 processes, the GPUs tile the first 4096*world batches of
    the EP sequence, and rank 0's processes cover exactly class A."""
    from paper_1511_07658_b200 import workloads as W
    sz = W.Sizes.for_world(world)
    assert (1 << (sz.ep_m - 16)) >= 4096 * world
    procs = 8
    cover = []
    for g in range(world):
        mine = [W.ep_slice("ep", g * procs + i, procs * world, sz) for i in range(procs)]
        assert sum(c for _, c in mine) == 4096
        assert mine[0][0] == 4096 * g
        cover += mine
    nxt = 0
    for first, count in cover:
        assert first == nxt and count == 512
        nxt += count
    # mixed: 4 EP workers per GPU (worker % 4 == 1), same tiling
    mixed = [W.ep_slice("mixed", w, 16 * world, sz) for w in range(16 * world) if w % 4 == 1]
    assert [f for f, _ in mixed] == [1024 * i for i in range(4 * world)]


def test_ep_verdict_rank0_class_a():
    a_sx, a_sy = R.NPB_EP_VERIFY[28]
    rank0 = R.empty_record()
    rank0[11], rank0[12], rank0[14] = a_sx, a_sy, 4096
    folded = R.empty_record()
    folded[11], folded[12], folded[14] = 2 * a_sx, 2 * a_sy, 8192
    v = R.ep_verdict(folded, 29, 8192, rank0)
    assert v["rank0_class_a_verified"] and v["verified"] and "npb_rel_err" not in v
    rank0[11] *= 1.0 + 1e-6
    assert not R.ep_verdict(folded, 29, 8192, rank0)["verified"]


def _rank_main_product(rank, world, port, path, out_q):
    """The product's bootstrap and fold (libvgpu.so through ctypes): GVM 0
    publishes the 128-byte NCCL id in a file, the others wait for it; the
    gathered records fold in rank order in C++ (vgpu_fold_in_rank_order)."""
    from paper_1511_07658_b200 import vgpu as V
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    if rank == 0:
        uid = bytes((i * 37 + 11) & 0xFF for i in range(128))  # stands in for ncclGetUniqueId
        V.rendezvous_publish(path, uid)
    else:
        uid = V.rendezvous_fetch(path, 128, timeout_ms=60000)
    workers = [2 * rank, 2 * rank + 1]
    results = [_worker_result(w, oracle.ep_job(24, 64 * w, 64)) for w in workers]
    rec = torch.tensor(R.record_from_workers(results), dtype=torch.float64)
    gathered = [torch.zeros_like(rec) for _ in range(world)]
    dist.all_gather(gathered, rec)
    flat = torch.cat(gathered).tolist()
    out_q.put((rank, uid, V.fold_in_rank_order(flat, world), R.fold_in_rank_order(flat, world)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_file_bootstrap_and_cpp_fold():
    import tempfile
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    path = os.path.join(tempfile.mkdtemp(), "ncclid")
    procs = [ctx.Process(target=_rank_main_product, args=(r, 2, port, path, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {r: rest for r, *rest in (q.get(timeout=240) for _ in procs)}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got[0][0] == got[1][0]  # every rank holds GVM 0's id
    for r in (0, 1):
        cpp, py = got[r][1], got[r][2]
        assert struct.pack("<15d", *cpp[:15]) == struct.pack("<15d", *py[:15])
    assert struct.pack("<16d", *got[0][1]) == struct.pack("<16d", *got[1][1])
    assert R.ep_verdict(got[0][1], 24)["verified"]
