"""Summarise a bench.py JSON line: python scripts/bsum.py gpurun_out/bench.log"""
import json
import sys

for line in open(sys.argv[1]):
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    if "roofline" not in d:
        print(d)
        continue
    print(f"value {d['value']:.4f} {d['unit']}  ms/step {d['ms_per_step']:.1f}  e2e {d['e2e']['value']}  launches {d['gpu_launches']}")
    print("roofline", {k: d["roofline"][k] for k in ("kernel", "achieved", "frac")})
    for k, v in d["roofline"]["live_kernels"].items():
        print(f"  {k:28s} n/step {v['launches_per_step']:7.0f} ms/step {v['ms_per_step']:8.2f} share {v['share_of_step']:.3f} us/launch {1e3*v['ms_per_launch']:9.1f} GB/s {v['achieved_gbs']:8.1f}")
    print("standalone", {k: round(v["achieved_gbs"]) for k, v in d["roofline"]["standalone_kernels"].items()})
    print("newton", d["newton"]["stats"], d["newton"]["setup_fgmres_ms_per_step"])
    print("cpu", d.get("cpu_baseline"))
