"""Summarize an .ncu-rep (raw page): key throughput, occupancy and stall metrics."""
import csv, subprocess, sys

KEYS = ['gpu__time_duration.sum', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__occupancy_limit_registers', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'smsp__warps_eligible.avg.per_cycle_active', 'smsp__warps_active.avg.per_cycle_active',
        'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum', 'l1tex__t_bytes.sum',
        'smsp__inst_executed.sum', 'smsp__sass_thread_inst_executed_op_fp64_pred_on.sum',
        'sm__cycles_elapsed.avg.per_second', 'launch__grid_size']

def main(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        print('---', vals[hdr.index('Kernel Name')][:60] if 'Kernel Name' in hdr else '')
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f'  {k:70s} {vals[i]:>16s} {units[i]}')
        st = []
        for i, h in enumerate(hdr):
            if h.startswith('smsp__pcsamp_warps_issue_stalled_') and not h.endswith('not_issued'):
                try:
                    v = float(vals[i].replace(',', ''))
                except ValueError:
                    continue
                if v > 0:
                    st.append((v, h.replace('smsp__pcsamp_warps_issue_stalled_', '')))
        tot = sum(v for v, _ in st) or 1
        print('  stalls:', ', '.join(f'{n} {100 * v / tot:.0f}%' for v, n in sorted(st, reverse=True)[:8]))

for p in sys.argv[1:]:
    print('=====', p)
    main(p)
