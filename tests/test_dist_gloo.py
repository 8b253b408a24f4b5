"""Multi-process (gloo, world_size 2, CPU) checks of the batch-sharding path.

Each rank runs its shard of the batch through the CPU oracle (the data path needs a GPU;
the host logic -- shard ranges, gathers, max-over-ranks timing, checksums -- does not) and
the gathered result must equal the unsharded run bit for bit.
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import oracle
    import synth
    from paper_1804_08378_b200 import dist as bsd

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        errors = []
        for wl in ("alexnet", "resnet50", "c1"):
            case = synth.workload(wl, batch=5)[0]
            N = case.shape[0]
            full = synth.uniform_np(case.input_seed, int(np.prod(case.shape))).reshape(case.shape)
            lo, hi = bsd.shard(N, world, rank)
            mine = oracle.run_bf(case.layers, full[lo:hi])
            got = bsd.gather_shards(torch.from_numpy(mine), N).numpy()
            ref = oracle.run_bf(case.layers, full)
            if not np.array_equal(got.view(np.uint32), ref.view(np.uint32)):
                errors.append(f"{wl}: gathered shards differ from the unsharded oracle run")
            sums = bsd.gather_stats([float(mine.astype(np.float64).sum()), float(rank)])
            if [int(s[1]) for s in sums] != list(range(world)):
                errors.append(f"gather_stats order {sums}")
            if abs(sum(s[0] for s in sums) - float(ref.astype(np.float64).sum())) > 1e-6 * max(1.0, abs(ref).sum()):
                errors.append("checksums do not add up")
        mx = bsd.max_over_ranks([float(rank) * 2.0, -float(rank)])
        if mx != [2.0 * (world - 1), 0.0]:
            errors.append(f"max_over_ranks {mx}")
        with open(os.path.join(out_dir, f"rank{rank}.txt"), "w") as f:
            f.write("\n".join(errors) if errors else "OK")
    finally:
        dist.destroy_process_group()


def test_shard_ranges():
    from paper_1804_08378_b200 import dist as bsd
    for n in (1, 5, 64, 128, 256, 257):
        for w in (1, 2, 3, 4, 8):
            rs = [bsd.shard(n, w, r) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
            sizes = [hi - lo for lo, hi in rs]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        bsd.shard(4, 2, 2)


def test_gloo_world_size_2():
    world = 2
    port = _free_port()
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, port, d), nprocs=world, join=True)
        for r in range(world):
            msg = open(os.path.join(d, f"rank{r}.txt")).read()
            assert msg == "OK", f"rank {r}: {msg}"
