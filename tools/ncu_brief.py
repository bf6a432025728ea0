"""Key metrics + top stall reasons of an ncu report (first kernel):
    ncu_brief.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, v = rows[0], rows[2]
d = dict(zip(h, v))
print(d.get("Kernel Name", "")[:120])
for k in ["gpu__time_duration.sum", "dram__bytes_read.sum",
          "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
          "l1tex__throughput.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
          "launch__registers_per_thread",
          "sm__warps_active.avg.pct_of_peak_sustained_active",
          "smsp__inst_executed.sum",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
          "smsp__sass_l1tex_data_pipe_lsu_wavefronts_mem_shared_op_ldgsts.sum",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
          "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_red.sum",
          "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum",
          "lts__t_sectors_srcunit_tex_op_red.sum",
          "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]:
    print(f"  {k:70s} {d.get(k)}")
st = [(k, d[k]) for k in h if k.startswith("smsp__average_warps_issue_stalled_")
      and k.endswith("_per_issue_active.ratio")]
st.sort(key=lambda x: -float(x[1] or 0))
print("  stalls per issue:", ", ".join(
    f"{k[34:-23]} {float(x):.2f}" for k, x in st[:8]))
