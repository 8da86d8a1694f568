"""Print selected raw ncu metrics per kernel: python tools/ncu_kv.py RAW.csv [substr...]"""
import csv, sys
r = list(csv.reader(open(sys.argv[1])))
h = r[0]; rows = r[2:]
ki = h.index('Kernel Name')
pats = ['gpu__time_duration.sum', 'smsp__inst_executed.sum', 'smsp__thread_inst_executed_per_inst_executed.ratio',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum', 'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum',
        'l1tex__t_sector_hit_rate.pct', 'lts__t_sector_hit_rate.pct', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'launch__registers_per_thread', 'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
        'sm__maximum_warps_per_active_cycle_pct', 'l1tex__throughput.avg.pct_of_peak_sustained_active']
stalls = [c for c in h if c.startswith('smsp__average_warps_issue_stalled_') and c.endswith('_per_issue_active.ratio')]
for row in rows:
    if len(sys.argv) > 2 and not any(s in row[ki] for s in sys.argv[2:]):
        continue
    print('==', row[ki][:70])
    for p in pats:
        if p in h:
            print('   %-70s %s' % (p, row[h.index(p)]))
    st = sorted(((float(row[h.index(c)] or 0), c) for c in stalls), reverse=True)[:7]
    print('   stalls:', ', '.join('%s %.2f' % (c[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')], v) for v, c in st))
