"""Host-side logic of the multi-GPU path on CPU: the communication plan of libdpd
(dpd_plan_peers) driven through a real multi-process exchange with torch.distributed
'gloo' (world size 2 and 4).  Every rank posts its sends/receives in increasing direction
index -- the order NCCL matches point-to-point operations in -- and each receive slot must
get the message its partner sent in that direction (halo and redistribution
messages to the adjacent ranks)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, grid, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1911_04712_b200 import capi
        to, fr, used = capi.dpd_plan_peers(grid, rank)
        reqs, bufs = [], {}
        for d in range(27):
            if not used[d]:
                continue
            msg = torch.tensor([rank, d, 1000 * rank + d], dtype=torch.int64)
            reqs.append(dist.isend(msg, int(to[d])))
            bufs[d] = torch.zeros(3, dtype=torch.int64)
            reqs.append(dist.irecv(bufs[d], int(fr[d])))
        for r in reqs:
            r.wait()
        ok = all(int(b[0]) == int(fr[d]) and int(b[1]) == d for d, b in bufs.items())
        # the messages a rank receives are exactly those its neighbours addressed to it
        q.put((rank, ok, sorted(bufs)))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:  # noqa: BLE001
        q.put((rank, False, repr(exc)))


@pytest.mark.parametrize("grid", [(2, 1, 1), (2, 2, 1), (1, 2, 2)])
def test_exchange_plan_pairs_messages(grid):
    world = grid[0] * grid[1] * grid[2]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, grid, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    # used directions: every nonzero component must be split
    for _, _, dirs in res:
        for d in dirs:
            D = (d % 3 - 1, (d // 3) % 3 - 1, d // 9 - 1)
            assert all(D[k] == 0 or grid[k] > 1 for k in range(3))


def test_plan_geometry():
    from paper_1911_04712_b200 import capi
    grid = (2, 2, 2)
    for rank in range(8):
        to, fr, used = capi.dpd_plan_peers(grid, rank)
        assert used.sum() == 26
        c = (rank % 2, (rank // 2) % 2, rank // 4)
        for d in range(27):
            D = (d % 3 - 1, (d // 3) % 3 - 1, d // 9 - 1)
            t = [(c[k] + D[k]) % 2 for k in range(3)]
            f = [(c[k] - D[k]) % 2 for k in range(3)]
            assert to[d] == t[0] + 2 * (t[1] + 2 * t[2])
            assert fr[d] == f[0] + 2 * (f[1] + 2 * f[2])
            # symmetry: the rank I send direction d to receives direction d from me
            to2, fr2, _ = capi.dpd_plan_peers(grid, int(to[d]))
            assert fr2[d] == rank
    to, fr, used = capi.dpd_plan_peers((2, 1, 1), 0)
    assert [d for d in range(27) if used[d]] == [12, 14]
