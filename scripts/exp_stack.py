"""Time one stack under several plan options (CUDA-graph bursts over rotating buffers).
usage: python scripts/exp_stack.py WORKLOAD IDX '{"force_generic":2}' '{}' ..."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_1804_08378_b200 as bs

peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
wl, idx = sys.argv[1], int(sys.argv[2])
optss = [(a if a == 'copy' else json.loads(a)) for a in sys.argv[3:]] or [{}]
case = synth.workload(wl)[idx]
dev = torch.device("cuda")
l2 = torch.cuda.get_device_properties(dev).L2_cache_size
res = []
for opts in optss:
    if opts == "copy":
        info0 = bs.bs_plan_query(bs.bs_plan_create(case.layers, case.shape, {"host_only": 1}))
        nb = info0["alg_bytes_read"] + info0["alg_bytes_written"]
        n = nb // 8
        nset = min(32, int(math.ceil(4 * l2 / nb)) + 1)
        bufs = [(torch.empty(n, device=dev), torch.empty(n, device=dev)) for q in range(nset)]
        R = max(8, min(64, 2 * nset))
        st = torch.cuda.Stream()
        def cburst():
            for r in range(R):
                x, y = bufs[r % nset]
                y.copy_(x)
        with torch.cuda.stream(st):
            cburst()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            cburst()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            g.replay(); a.record(st)
            for _ in range(5): g.replay()
            b.record(st)
        torch.cuda.synchronize()
        t = a.elapsed_time(b) / (5 * R)
        print(json.dumps({"stack": case.name, "opts": "torch copy_ same bytes", "kernel": "copy", "us": t * 1e3,
                          "gbs": nb / (t / 1e3) / 1e9, "frac": nb / (t / 1e3) / 1e9 / peak, "grid": 0, "tasks": 0,
                          "rows": 0, "G": 0, "J": 0}), flush=True)
        continue
    plan = bs.bs_plan_create(case.layers, case.shape, opts or None)
    info = bs.bs_plan_query(plan)
    nb = info["alg_bytes_read"] + info["alg_bytes_written"]
    nset = min(32, int(math.ceil(4 * l2 / nb)) + 1)
    bufs = [(synth.uniform_torch(case.input_seed + q, case.shape, device=dev), torch.empty(info["out"], device=dev))
            for q in range(nset)]
    R = max(8, min(64, 2 * nset))
    def burst(sh):
        for r in range(R):
            x, y = bufs[r % nset]
            bs.bs_execute(plan, x.data_ptr(), y.data_ptr(), sh)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        burst(st.cuda_stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        burst(torch.cuda.current_stream().cuda_stream)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        g.replay()
        a.record(st)
        for _ in range(5):
            g.replay()
        b.record(st)
    torch.cuda.synchronize()
    t = a.elapsed_time(b) / (5 * R)
    li = bs.bs_plan_query_launch(plan, 0)
    r = {"stack": case.name, "opts": opts, "kernel": bs.KERNEL_NAMES[li["kernel"]], "us": t * 1e3,
         "gbs": nb / (t / 1e3) / 1e9, "frac": nb / (t / 1e3) / 1e9 / peak, "grid": li["grid"], "tasks": li["n_tasks"],
         "rows": li["rows_per_task"], "G": li["groups_per_warp"], "J": li["outputs_per_group"]}
    res.append(r)
    print(json.dumps(r), flush=True)
    del bufs, g
