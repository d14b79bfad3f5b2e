"""Summarise an ncu report: per-kernel duration, DRAM bytes, occupancy, top stalls."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
want = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__occupancy_limit_shared_mem',
        'launch__occupancy_limit_registers', 'launch__registers_per_thread', 'smsp__inst_executed.sum']
units = rows[1]
for r in rows[2:]:
    name = r[hdr.index('Kernel Name')].split('(')[0][-24:]
    st = [(hdr[i].replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''), float(r[i]))
          for i in range(len(hdr)) if hdr[i].startswith('smsp__average_warps_issue_stalled_')
          and hdr[i].endswith('per_issue_active.ratio') and r[i] not in ('', 'n/a')]
    st.sort(key=lambda x: -x[1])
    print(name, ' '.join(w.split('__')[-1][:20] + '=' + r[hdr.index(w)] + units[hdr.index(w)] for w in want if w in hdr))
    print('     stalls', [(a, round(b, 2)) for a, b in st[:6]])
