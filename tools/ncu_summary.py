"""Summarise ncu reports into profiles/ text files (dev aid)."""
import csv, io, subprocess, sys
KEYS = ['gpu__time_duration.sum', 'sm__cycles_elapsed.avg.per_second', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__shared_mem_per_block_dynamic', 'launch__grid_size',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem', 'smsp__inst_executed.sum',
        'smsp__sass_inst_executed_op_local_ld.sum', 'smsp__sass_inst_executed_op_local_st.sum']
for rep in sys.argv[1:]:
    raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    hdr, units = r[0], r[1]
    for row in r[2:]:
        d = dict(zip(hdr, row)); u = dict(zip(hdr, units))
        print(f"== {d.get('Kernel Name','')[:80]}  ({rep.split('/')[-1]})")
        for k in KEYS:
            if k in d:
                print(f"  {k:62s} {d[k]:>18s} {u.get(k,'')}")
        st = [(float(d[k].replace(',', '')), k) for k in hdr if 'issue_stalled' in k and k.endswith('per_issue_active.ratio')
              and d.get(k, '') not in ('', 'n/a')]
        for v, k in sorted(st, reverse=True)[:6]:
            print(f"  stall {k.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio',''):30s} {v:8.3f}")
