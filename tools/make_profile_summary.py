"""Writes profiles/ncu_summary.json and profiles/<round>_ncu.md from .ncu-rep
captures (run in the build container: `ncu -i` works without a GPU)."""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    'time_us': ('gpu__time_duration.sum', 1e-3),
    'dram_read_bytes': ('dram__bytes_read.sum', None),
    'dram_write_bytes': ('dram__bytes_write.sum', None),
    'dram_pct_peak': ('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', None),
    'tensor_active_pct': ('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed', None),
    'sm_throughput_pct': ('sm__throughput.avg.pct_of_peak_sustained_elapsed', None),
    'l2_throughput_pct': ('lts__throughput.avg.pct_of_peak_sustained_elapsed', None),
    'xbar2l1_bytes': ('l1tex__m_xbar2l1tex_read_bytes.sum', None),
    'sm_clock_ghz': ('sm__cycles_elapsed.avg.per_second', None),
    'registers': ('launch__registers_per_thread', None),
    'grid': ('launch__grid_size', None),
    'warps_active_pct': ('sm__warps_active.avg.pct_of_peak_sustained_active', None),
}
SCALE = {'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'Tbyte': 1e12, 'byte': 1, 'ms': 1e3, 'us': 1, 'ns': 1e-3,
         'Ghz': 1, 'Mhz': 1e-3}


def read(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    res = {'kernel': vals[hdr.index('Kernel Name')][:120]}
    for key, (m, _) in METRICS.items():
        if m in hdr:
            i = hdr.index(m)
            v = float(vals[i].replace(',', ''))
            u = units[i]
            if key == 'time_us':
                v = v * SCALE.get(u, 1)
            elif u in SCALE and 'byte' in u.lower():
                v = v * SCALE[u]
            res[key] = v
    return res


def main():
    rnd = sys.argv[1]
    caps = dict(a.split('=', 1) for a in sys.argv[2:])
    summary = {}
    lines = [f"# ncu --set full captures, {rnd} (clock-control none; per-launch values)\n",
             "| capture | kernel | time µs | DRAM read | DRAM write | DRAM %pk | tensor % | L2 % | L2->SM bytes | SM GHz | regs | grid |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for name, path in caps.items():
        r = read(path)
        summary[name] = r
        lines.append(f"| {name} | `{r['kernel'][:50]}` | {r.get('time_us', 0):.1f} | {r.get('dram_read_bytes', 0)/1e9:.3f} GB | "
                     f"{r.get('dram_write_bytes', 0)/1e9:.3f} GB | {r.get('dram_pct_peak', 0):.1f} | {r.get('tensor_active_pct', 0):.1f} | "
                     f"{r.get('l2_throughput_pct', 0):.1f} | {r.get('xbar2l1_bytes', 0)/1e9:.2f} GB | {r.get('sm_clock_ghz', 0):.2f} | "
                     f"{int(r.get('registers', 0))} | {int(r.get('grid', 0))} |")
    js = {}
    for name, r in summary.items():
        js[name] = dict(r, dram_bytes_per_launch=r.get('dram_read_bytes', 0) + r.get('dram_write_bytes', 0))
    # bench.py looks up its dominant kernel under these keys
    if 'ag_cfg2' in js:
        js['ag_gemm_sm100_kernel'] = js['ag_cfg2']
    with open('profiles/ncu_summary.json', 'w') as f:
        json.dump(js, f, indent=1)
    with open(f'profiles/{rnd}_ncu.md', 'w') as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == '__main__':
    main()
