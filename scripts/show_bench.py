import glob, json, sys
for f in sorted(glob.glob(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/bench*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f"{f:40s} {d['value']/1e6:8.2f}M e2e {d['e2e']['value']/1e6:8.2f}M  {d['ms_per_step']:.3f} ms  N={d['config'].get('rollouts_per_step_per_gpu')}  frac={d['roofline']['frac']:.3f} clk={d['clocks'].get('sm_mhz')}/{d['clocks'].get('samples')}")
    except Exception as e:
        print(f, "ERR", e)
