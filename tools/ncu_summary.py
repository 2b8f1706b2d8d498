"""Summarise an ncu report (raw page) for the metrics that matter here."""
import csv
import subprocess
import sys

WANT = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__inst_executed.sum',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__t_bytes.sum', 'lts__t_bytes.sum',
        'launch__block_size', 'launch__grid_size']


def main(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    stall = [h for h in hdr if h.startswith('smsp__pcsamp_warps_issue_stalled') and not h.endswith('not_issued')]
    for row in rows[2:]:
        print('---')
        for w in WANT:
            if w in hdr:
                print(f'{w} = {row[hdr.index(w)][:90]}')
        vals = []
        for h in stall:
            try:
                vals.append((float(row[hdr.index(h)]), h.split('stalled_')[-1]))
            except ValueError:
                pass
        vals.sort(reverse=True)
        tot = sum(v for v, _ in vals) or 1
        print('stalls:', ', '.join(f'{n} {100 * v / tot:.0f}%' for v, n in vals[:8]))


if __name__ == '__main__':
    main(sys.argv[1])
