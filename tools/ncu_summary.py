"""Summarise an .ncu-rep (raw page + source page) into the metrics we track."""
import csv, subprocess, sys, collections, io, json

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'dram__cycles_active.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__occupancy_limit_registers', 'sm__maximum_warps_per_active_cycle_pct',
        'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum', 'l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum',
        'l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum', 'l1tex__t_requests_pipe_lsu_mem_global_op_st.sum',
        'lts__t_sectors_srcunit_tex_op_read.sum', 'lts__t_sectors_srcunit_tex_op_write.sum',
        'lts__t_sector_hit_rate.pct', 'l1tex__t_sector_hit_rate.pct',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed', 'l1tex__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__data_pipe_lsu_wavefronts.sum', 'lts__t_sectors_op_read.sum', 'lts__t_sectors_op_write.sum',
        'dram__sectors_read.sum', 'dram__sectors_write.sum', 'launch__grid_size', 'launch__block_size',
        'smsp__cycles_active.avg', 'sm__cycles_elapsed.max']

def raw(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {'kernel': r[hdr.index('Kernel Name')]}
        for w in WANT:
            if w in hdr:
                d[w] = (r[hdr.index(w)], units[hdr.index(w)])
        res.append(d)
    return res

def source(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    iS, iE = hdr.index('Source'), hdr.index('Instructions Executed')
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith('stall_') and 'Not Issued' not in h]
    ops, stall, tot, n = collections.Counter(), collections.Counter(), 0, 0
    for r in rows[2:]:
        if r and r[0] == 'Kernel Name':
            break
        if len(r) < len(hdr):
            continue
        toks = r[iS].split()
        op = toks[1] if toks[0].startswith('@') else toks[0]
        op = op.split('.')[0] + ('.128' if '.128' in r[iS] else '.64' if ('.64 ' in r[iS] and op[:3] in ('LDG','STG')) else '')
        e = int(r[iE]); ops[op] += e; tot += e; n += 1
        for i in stall_cols:
            stall[hdr[i]] += int(r[i])
    return ops, stall, tot, n

if __name__ == '__main__':
    path = sys.argv[1]
    cells = float(sys.argv[2]) if len(sys.argv) > 2 else 512.0 ** 3
    for d in raw(path)[:1]:
        print('kernel:', d['kernel'])
        for k, v in d.items():
            if k != 'kernel':
                print(f'  {k:72s} {v[0]:>18s} {v[1]}')
    ops, stall, tot, n = source(path)
    print(f'static SASS instructions {n}; executed warp-instructions {tot} = {tot / cells:.2f} per cell')
    for op, c in ops.most_common(16):
        print(f'  {op:12s} {c / cells:8.3f} per cell')
    s = sum(stall.values())
    print('stalls:', ', '.join(f'{k[6:]} {100 * v / s:.1f}%' for k, v in stall.most_common(8)))
