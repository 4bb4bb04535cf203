"""Summarise an .ncu-rep: key metrics + top stall sites (run here, no GPU)."""
import csv
import io
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'launch__registers_per_thread', 'launch__grid_size', 'launch__occupancy_limit_registers',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__occupancy_per_block_size',
        'sm__maximum_warps_per_active_cycle_pct', 'launch__waves_per_multiprocessor',
        'smsp__inst_executed.sum', 'sm__cycles_elapsed.avg.per_second', 'l1tex__throughput.avg.pct_of_peak_sustained_active']


def raw(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2]


def main(path, top=12):
    hdr, units, vals = raw(path)
    res = {}
    for k in KEYS:
        for i, h in enumerate(hdr):
            if h == k or (h.startswith(k) and k.endswith('pct_of_peak_sustained_elapsed') is False and h == k):
                res[h] = (vals[i], units[i])
    for i, h in enumerate(hdr):
        if h in KEYS:
            print(f"{h:70s} {vals[i]:>14s} {units[i]}")
    stalls = []
    for i, h in enumerate(hdr):
        if h.startswith('smsp__pcsamp_warps_issue_stalled_') and not h.endswith('not_issued'):
            try:
                stalls.append((float(vals[i]), h.replace('smsp__pcsamp_warps_issue_stalled_', '')))
            except ValueError:
                pass
    tot = sum(s for s, _ in stalls) or 1
    print("stalls:", ", ".join(f"{n} {100*s/tot:.0f}%" for s, n in sorted(stalls, reverse=True)[:8]))
    out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if 'Warp Stall Sampling (All Samples)' in r)
    hdr = rows[hi]
    si = hdr.index('Warp Stall Sampling (All Samples)')
    src = hdr.index('Source')
    data = []
    for r in rows[hi + 1:]:
        try:
            data.append((int(r[si]), r[src]))
        except (ValueError, IndexError):
            pass
    t = sum(d[0] for d in data) or 1
    for n, s in sorted(data, reverse=True)[:top]:
        print(f"  {100*n/t:5.1f}%  {s[:110]}")


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 12)
