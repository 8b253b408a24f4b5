"""torchrun worker for tests/test_bench_dist.py: bench.py's multi-rank host logic (aggregate,
shard ranges, gathered-shard validation) with a stub executor on CPU (gloo).  Not a test file."""
import fcntl
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1804_08378_b200 import dist as bsd  # noqa: E402
from tests import _util as U  # noqa: E402


def main():
    out_dir = sys.argv[1]
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    res = {}
    # ---- timing: a stub "device" shared by both ranks (an exclusive lock), 4 steps of 0.1 s each
    lock_path = os.path.join(out_dir, "device.lock")
    steps, t_step = 4, 0.1

    def stub_step():
        with open(lock_path, "a") as f:
            fcntl.flock(f, fcntl.LOCK_EX)
            t0 = time.perf_counter()
            time.sleep(t_step)
            fcntl.flock(f, fcntl.LOCK_UN)
        return time.perf_counter() - t0

    for shared in (True, False):
        dist.barrier()
        w0 = time.perf_counter()
        dev_s = 0.0
        for _ in range(steps):
            if shared:
                dev_s += stub_step()              # serialised with the other rank
            else:
                time.sleep(t_step)                # a device of its own
                dev_s += t_step
        dist.barrier()
        wall = time.perf_counter() - w0
        agg = bench.aggregate(8, 1e3 * dev_s, wall, steps, "cpu")
        res["shared" if shared else "own"] = agg
    # ---- validation of gathered shards (strong and weak layouts)
    case = synth.workload("alexnet", batch=1)[0]
    for strong in (True, False):
        n_full = 5
        lo, hi = bench.shard_of(n_full, world, rank, strong)
        n_total = n_full if strong else n_full * world
        chw = int(np.prod(case.shape[1:]))
        shp = (hi - lo,) + tuple(case.shape[1:])
        x = synth.uniform_np(case.input_seed, (hi - lo) * chw, start=lo * chw).reshape(shp)
        y = torch.from_numpy(oracle.run_bf(case.layers, x))          # the stub executor
        if rank == 1 and not strong:
            y[0, 0, 0, 0] += 1.0                                     # a corrupted shard must be caught
        g = bsd.gather_shards(y, n_total, "cpu")

        def ref_image(n):
            xi = synth.uniform_np(case.input_seed, chw, start=n * chw).reshape((1,) + tuple(case.shape[1:]))
            return oracle.run_bf(case.layers, xi)
        v = bench.validate_gathered(g.numpy(), n_total, ref_image,
                                    lambda got, ref, c: U.check(got, ref, case.layers, c), samples=n_total)
        res["strong" if strong else "weak"] = {"n_total": n_total, "gathered": int(g.shape[0]), **v}
    json.dump(res, open(os.path.join(out_dir, f"rank{rank}.json"), "w"))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
