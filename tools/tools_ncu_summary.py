import csv, gzip, sys
d_ = sys.argv[1]
rows = list(csv.reader(open(f'{d_}/details.csv')))
hdr = rows[0]; idx = {h:i for i,h in enumerate(hdr)}
want = ['Duration','DRAM Throughput','Memory Throughput','L1/TEX Hit Rate','L2 Hit Rate','Achieved Occupancy','Registers Per Thread','Compute (SM) Throughput','L1/TEX Cache Throughput','L2 Cache Throughput','Executed Ipc Active','Block Limit Registers','Mem Busy','Max Bandwidth','Mem Pipes Busy']
for r in rows[1:]:
    if r[idx['ID']] != '0': continue
    if r[idx['Metric Name']] in want: print(r[idx['Metric Name']], r[idx['Metric Value']], r[idx['Metric Unit']])
print(rows[1][idx['Kernel Name']][:80])
rows = list(csv.reader(gzip.open(f'{d_}/raw.csv.gz','rt')))
d = {h:v for h,v in zip(rows[0], rows[2])}
def f(v):
    try: return float(v.replace(',',''))
    except: return None
st = sorted([(f(v), h) for h,v in d.items() if 'pcsamp_warps_issue_stalled' in h and not h.endswith('not_issued') and f(v) is not None], reverse=True)[:8]
for s,h in st: print('STALL', h.replace('smsp__pcsamp_warps_issue_stalled_',''), s)
for h in ['l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum','l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum','lts__t_sectors_srcunit_tex_op_read.sum','dram__bytes_read.sum','dram__bytes_write.sum','smsp__inst_executed.sum','l1tex__data_pipe_lsu_wavefronts.sum','l1tex__data_pipe_lsu_wavefronts_mem_lg.sum','l1tex__t_sector_hit_rate.pct','sm__warps_active.avg.pct_of_peak_sustained_active']:
    print(h, d.get(h))
