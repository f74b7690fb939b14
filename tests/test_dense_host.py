"""Host logic of the tile-cyclic dense Cholesky (BASELINE config 4), on CPU.

The multi-GPU path (paper_2008_01541_b200/dense.py, csrc/dense_ctx.cu) has
no collective on its data path: each rank runs the tile tasks it owns, in the
global claim order, and waits on per-tile flags that the owners of the
producing tiles release. What must hold on the host side:

* the ranks' task lists partition the single-GPU task list, each one a
  subsequence of the global claim order, with the ownership rule of
  `dense_tile_owner` (column-cyclic; a sub-diagonal partial goes with the
  diagonal that finalizes it);
* with the kernel's dependency rules and a bounded number of CTAs per rank
  claiming in order, the schedule always completes (no cross-rank deadlock);
* the IPC-handle exchange over torch.distributed returns every rank's handle
  in rank order (world_size-2 gloo group).

Nothing here touches a GPU: `spb_dense_rank_tasks` is host-only.
"""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2008_01541_b200 import dense  # noqa: E402
from paper_2008_01541_b200.errors import InvalidArgumentError  # noqa: E402


def _pairs(a):
    return [tuple(map(int, t)) for t in a]


@pytest.mark.parametrize("m", [64, 200, 1000, 3000])
@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_rank_tasks_partition_global_order(m, P):
    glob = _pairs(dense.rank_tasks(m, 0, 1))
    N = (m + 63) // 64
    assert len(glob) == N * (N + 1) // 2
    pos = {t: k for k, t in enumerate(glob)}
    seen = set()
    for r in range(P):
        mine = _pairs(dense.rank_tasks(m, r, P))
        order = [pos[t] for t in mine]
        assert order == sorted(order), "a rank's tasks must keep the global claim order"
        for (i, j) in mine:
            assert dense.tile_owner(i, j, P) == r
            assert (i, j) not in seen
            seen.add((i, j))
    assert seen == set(glob)


def _deps(i, j):
    """Tiles a task waits on, with the flag value it needs (dense.cu
    cholesky_body): 'F' = final tile, 'P' = published partial, 'D' = diagonal
    factor (L_jj^-T) of that column."""
    out = []
    if i == j:
        out += [("F", j, k) for k in range(j - 1)]
        if j > 0:
            out += [("P", j, j - 1), ("D", j - 1, j - 1)]
    else:
        for k in range(j):
            out += [("F", i, k), ("F", j, k)]
        if i != j + 1:
            out.append(("D", j, j))
    return out


def _simulate(m, P, ctas_per_rank):
    """Each rank: `ctas_per_rank` workers claim its tasks in order; a claimed
    task finishes once its dependencies are done. Returns rounds or raises."""
    N = (m + 63) // 64
    lists = [_pairs(dense.rank_tasks(m, r, P)) for r in range(P)]
    nxt = [0] * P
    running = [[] for _ in range(P)]
    done = set()
    total = sum(len(x) for x in lists)
    finished = 0
    rounds = 0
    while finished < total:
        rounds += 1
        for r in range(P):
            while len(running[r]) < ctas_per_rank and nxt[r] < len(lists[r]):
                running[r].append(lists[r][nxt[r]])
                nxt[r] += 1
        completed = []
        for r in range(P):
            for t in running[r]:
                if all(d in done for d in _deps(*t)):
                    completed.append((r, t))
        if not completed:
            raise AssertionError(f"deadlock: m={m} P={P} ctas={ctas_per_rank} after {finished}/{total}")
        for r, (i, j) in completed:
            running[r].remove((i, j))
            finished += 1
            if i == j:
                done.add(("D", j, j))
                if j > 0:
                    done.add(("F", j, j - 1))  # the diagonal task finalizes the partial
            elif i == j + 1:
                done.add(("P", i, j))
            else:
                done.add(("F", i, j))
    assert N >= 1
    return rounds


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_schedule_completes_with_resident_ctas(P):
    # 148 SMs: 148 // P CTAs per rank on one GPU each is the real case; the
    # emulated mode gives each rank ~148 / P CTAs of one GPU, and a small
    # worker count is the stress case for the lead-ahead diagonal claims
    for m in (640, 2000):
        for ctas in (6, max(6, 148 // P)):
            _simulate(m, P, ctas)


def test_rank_tasks_rejects_bad_arguments():
    with pytest.raises(InvalidArgumentError):
        dense.rank_tasks(100, 2, 2)
    with pytest.raises(InvalidArgumentError):
        dense.rank_tasks(100, 0, 9)
    with pytest.raises(InvalidArgumentError):
        dense.rank_tasks(0, 0, 1)


def test_gather_handles_validates():
    h = [bytes([r]) * dense.IPC_BYTES for r in range(3)]
    got = dense.gather_handles(h[1], 1, 3, lambda obj: [(2, h[2]), (0, h[0]), obj])
    assert got == h
    with pytest.raises(InvalidArgumentError):
        dense.gather_handles(b"short", 0, 1, lambda obj: [obj])
    with pytest.raises(InvalidArgumentError):
        dense.gather_handles(h[0], 0, 2, lambda obj: [obj, obj])  # duplicate rank


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        local = bytes([17 * (rank + 1)]) * dense.IPC_BYTES
        got = dense.gather_handles(local, rank, world, dense._dist_all_gather())
        np.save(Path(out_dir) / f"h{rank}.npy", np.frombuffer(b"".join(got), dtype=np.uint8))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_handle_exchange_gloo_world2(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    want = np.frombuffer(b"".join(bytes([17 * (r + 1)]) * dense.IPC_BYTES for r in range(world)), dtype=np.uint8)
    for r in range(world):
        assert np.array_equal(np.load(tmp_path / f"h{r}.npy"), want)
