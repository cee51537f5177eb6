"""Summarise an ncu report: key throughput counters (raw page) and top stall lines (source page)."""
import csv, io, subprocess, sys
KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_tensor', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed', 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'lts__t_sectors_srcunit_tex_op_read.sum', 'lts__t_bytes.sum', 'smsp__inst_executed.sum',
        'sm__cycles_elapsed.avg', 'launch__grid_size', 'launch__registers_per_thread',
        'smsp__average_warp_latency_issue_stalled', 'l1tex__m_xbar2l1tex_read_bytes.sum',
        'sm__memory_throughput.avg.pct', 'lts__t_sectors_op_read.sum', 'lts__t_sectors_op_write.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared']
def raw(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = {}
    for k in KEYS:
        for i, h in enumerate(hdr):
            if h.startswith(k) and not h.endswith('.per_second') and 'peak_sustained_elapsed.per' not in h:
                res[h] = (units[i], [r[i] for r in data])
    return res
def source(rep, top=20):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]; data = rows[2:]
    i_s = hdr.index("Warp Stall Sampling (Not-issued Samples)"); i_src = hdr.index("Source")
    data = [r for r in data if len(r) > i_s and r[i_s].isdigit()]
    tot = sum(int(r[i_s]) for r in data)
    return tot, [(int(r[i_s]), r[i_src].strip()[:80]) for r in sorted(data, key=lambda r: -int(r[i_s]))[:top]]
if __name__ == '__main__':
    for rep in sys.argv[1:]:
        print('==', rep)
        for k, (u, v) in raw(rep).items():
            print(f'  {k} [{u}] {v}')
        tot, top = source(rep)
        print('  not-issued stall samples', tot)
        for n, src in top:
            print(f'   {n:6d} {src}')
