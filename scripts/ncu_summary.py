"""Summarise ncu reports (run here, no GPU needed): key counters per kernel."""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "duration_us": ("gpu__time_duration.sum", 1e-3),
    "dram_read_MB": ("dram__bytes_read.sum", None),
    "dram_write_MB": ("dram__bytes_write.sum", None),
    "dram_pct_peak": ("dram__throughput.avg.pct_of_peak_sustained_elapsed", None),
    "smem_ld_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", None),
    "smem_st_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", None),
    "smem_ld_inst": ("smsp__sass_inst_executed_op_shared_ld.sum", None),
    "smem_st_inst": ("smsp__sass_inst_executed_op_shared_st.sum", None),
    "smem_ld_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", None),
    "smem_st_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", None),
    "shfl_inst": ("smsp__sass_inst_executed_op_shfl.sum", None) ,
    "inst_executed": ("smsp__inst_executed.sum", None),
    "regs": ("launch__registers_per_thread", None),
    "grid": ("launch__grid_size", None),
    "block": ("launch__block_size", None),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", None),
    "gld_sectors": ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", None),
    "gld_requests": ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", None),
    "gst_sectors": ("l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", None),
    "gst_requests": ("l1tex__t_requests_pipe_lsu_mem_global_op_st.sum", None),
}


def summarize(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {"report": rep, "kernel": vals[hdr.index("Kernel Name")][:120]}
    for k, (m, _) in KEYS.items():
        if m in hdr:
            v = vals[hdr.index(m)].replace(",", "")
            u = units[hdr.index(m)]
            try:
                x = float(v)
            except ValueError:
                d[k] = v
                continue
            if u == "Gbyte":
                x *= 1000
            elif u == "Kbyte":
                x /= 1000
            elif u == "byte":
                x /= 1e6
            elif u == "ms":
                x *= 1000
            elif u == "ns" and k == "duration_us":
                x /= 1000
            d[k] = x
    if d.get("smem_ld_inst"):
        d["smem_ld_wavefronts_per_inst"] = d["smem_ld_wavefronts"] / d["smem_ld_inst"]
    if d.get("smem_st_inst"):
        d["smem_st_wavefronts_per_inst"] = d["smem_st_wavefronts"] / d["smem_st_inst"]
    if d.get("gld_requests"):
        d["gld_sectors_per_request"] = d["gld_sectors"] / d["gld_requests"]
    if d.get("gst_requests"):
        d["gst_sectors_per_request"] = d["gst_sectors"] / d["gst_requests"]
    return d


if __name__ == "__main__":
    res = [summarize(r) for r in sys.argv[1:]]
    print(json.dumps(res, indent=1))
