"""Summarise an ncu --set full report: key throughput metrics + top stall reasons."""
import csv, io, json, subprocess, sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread', 'launch__grid_size',
        'launch__block_size', 'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
        'lts__t_bytes.sum', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__m_xbar2l1tex_read_bytes.sum', 'sm__memory_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__sass_thread_inst_executed_op_fadd_pred_on.sum']


def summarise(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        m = {k: (d.get(k), units[hdr.index(k)]) for k in KEYS if k in hdr}
        st = {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''): float(d[k])
              for k in hdr if 'smsp__average_warps_issue_stalled' in k and k.endswith('ratio')
              and d[k] not in ('', 'n/a') and float(d[k]) > 0.05}
        res.append({'kernel': d.get('Kernel Name'), 'metrics': m,
                    'stalls': dict(sorted(st.items(), key=lambda kv: -kv[1]))})
    return res


if __name__ == '__main__':
    r = summarise(sys.argv[1])
    if len(sys.argv) > 2:
        json.dump({'report': sys.argv[1], 'launches': r}, open(sys.argv[2], 'w'), indent=1)
    for x in r:
        print(x['kernel'][:80])
        for k, v in x['metrics'].items():
            print(f"  {k:70s} {v[0]} {v[1]}")
        print('  stalls:', x['stalls'])
