"""Summarise an ncu report: key SOL metrics per kernel + top stall reasons + hottest SASS."""
import csv, collections, subprocess, sys, io
rep = sys.argv[1]
want = ['Duration', 'Elapsed Cycles', 'DRAM Throughput', 'Memory Throughput', 'L2 Cache Throughput', 'L1/TEX Cache Throughput',
        'Executed Ipc Active', 'Issue Slots Busy', 'Registers Per Thread', 'Block Size', 'Grid Size', 'Cluster Size',
        'Achieved Occupancy', 'Warp Cycles Per Issued Instruction', 'Executed Instructions', 'One or More Eligible']
out = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
seen = collections.OrderedDict()
for r in rows[1:]:
    d = dict(zip(hdr, r))
    key = (d['ID'], d['Kernel Name'][:60])
    if d['Metric Name'] in want:
        seen.setdefault(key, {})[d['Metric Name']] = d['Metric Value'] + ' ' + d['Metric Unit']
for k, v in seen.items():
    print('==', k)
    for m in want:
        if m in v: print('   ', m.ljust(36), v[m])
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h = rr[0]
for r in rr[2:]:
    d = dict(zip(h, r))
    print('== raw', d.get('ID'), d.get('Kernel Name', '')[:40], 'dram_rd', d.get('dram__bytes_read.sum'), 'dram_wr', d.get('dram__bytes_write.sum'),
          'lts_rd', d.get('lts__t_bytes_srcunit_tex_op_read.sum'), 'time', d.get('gpu__time_duration.sum'))
