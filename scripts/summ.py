import json, sys
for l in open(sys.argv[1]):
    d=json.loads(l)
    r=d['roofline']; lbl=d.get('layer_by_layer_torch') or {}
    print(f"{d['config']['workload']:12s} ips={d['value']:10.0f} ms={d['ms_per_step']:.4f} step={d['hbm']['alg_gbs_per_gpu']:6.0f}GB/s ({d['hbm']['pct_of_measured_peak']:5.1f}%) dom={r['stack']:28s} {r['achieved']:6.0f}GB/s frac={r['frac']:.3f} dom_ms={r['avg_launch_ms']:.4f} e2e={d['e2e']['value']:.0f} lbl_x={lbl.get('fused_speedup',0):.2f} clk={d['clocks']['sm_mhz']}")
    for p in d.get('per_stack') or []:
        print(f"    {p['stack']:34s} x{p['count']:<3d} {str(tuple(p['shape'])):22s} {p['kernel']:20s} {p['ms']*1e3:8.1f}us {p['gbs']:6.0f}GB/s {p['frac']:.3f}")
