"""Key ncu metrics per captured kernel (from a --set full report): time, issue, smem wavefronts,
occupancy, DRAM bytes, L2/L1 throughput.  usage: python tools/ncu_summary.py <rep.ncu-rep>"""
import csv, io, subprocess, sys
M = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg", "smsp__issue_active.avg.pct_of_peak_sustained_active",
     "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
     "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
     "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "launch__registers_per_thread",
     "l1tex__throughput.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--metrics", ",".join(M)],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[0]
for row in r[2:]:
    d = dict(zip(h, row))
    f = lambda k: float(d[k].replace(",", "")) if d.get(k) not in (None, "", "n/a") else float("nan")
    cyc = f("sm__cycles_elapsed.avg")
    print(f"{d['Kernel Name'][:38]:38s} t={f('gpu__time_duration.sum')/1e3:8.1f}us issue={f('smsp__issue_active.avg.pct_of_peak_sustained_active'):5.1f}% "
          f"inst={f('smsp__inst_executed.sum')/1e6:7.1f}M smem_wf/clk/SM={f('l1tex__data_pipe_lsu_wavefronts_mem_shared.sum')/cyc/148:5.2f} "
          f"conf={f('l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum')/1e6:6.2f}M warps={f('sm__warps_active.avg.pct_of_peak_sustained_active'):5.1f}% "
          f"dram={(f('dram__bytes_read.sum')+f('dram__bytes_write.sum'))/1e6:7.1f}MB L2={f('lts__t_bytes.sum')/1e6:8.1f}MB l1={f('l1tex__throughput.avg.pct_of_peak_sustained_active'):5.1f}% "
          f"regs={d.get('launch__registers_per_thread')} grid={d.get('launch__grid_size')} blk={d.get('launch__block_size')}")
