"""One-screen summary of a bench.py JSON line: python tools/bench_summary.py FILE"""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(f"headline {d['value']:.1f} us  frac {d['roofline']['frac']:.3f}  bsp {d['bsp']['value']:.1f}  "
      f"e2e {d['e2e']['value']:.1f}  clocks {d['clocks'].get('sm_mhz')} {d['clocks'].get('violation_ms')}  "
      f"launches {d.get('gpu_launches')}  num {d['numerics']['ag_sampled_rows_norm_err']:.2e}")
for k in ("fd_config3_b1_L128k", "fd_config4_b32_L32k"):
    s = d["secondary"][k]
    print(f"{k}: fused {s['fused_us']:.1f} f32 {s['fused_f32out_us']:.1f} bsp {s['bsp_us']:.1f} "
          f"nccl {s['nccl_bsp_us']:.1f} graph {s.get('bsp_cuda_graph_us', 0):.1f} frac {s['roofline']['frac']:.3f} "
          f"e2e {s.get('e2e', {}).get('value', 0):.1f} num {s['numerics']['bf16']['head_rel_err']:.2e}/"
          f"{s['numerics']['f32']['head_rel_err']:.2e} cpu {s.get('cpu_baseline', {}).get('value', 0) / 1e6:.2f}s")
for m, p in d["secondary"]["ag_msweep_K8192_N8192"]["points"].items():
    print(f"  M={m:>6} best {p['best']} {p[p['best']]['mean_us']:9.1f} us  bsp {p['bsp']['mean_us']:9.1f}  "
          f"x{p['fused_speedup_vs_bsp']:.2f}  frac {p['roofline']['frac']:.3f} ({p['roofline']['bound']})")
