"""L1 data-pipe wavefront breakdown of an ncu report (shared / global ld / global st)."""
import csv
import io
import subprocess
import sys

for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    v = dict(zip(r[0], r[2]))

    def g(k):
        try:
            return float(v[k].replace(",", ""))
        except (KeyError, ValueError):
            return float("nan")
    print(rep)
    for k in ("gpu__time_duration.sum", "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
              "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum",
              "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_st.sum",
              "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
              "l1tex__lsuin_requests.sum.pct_of_peak_sustained_elapsed",
              "l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum", "smsp__inst_executed.sum"):
        print(f"  {k:70s} {g(k):.4g}")
