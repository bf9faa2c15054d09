"""Summarise an ncu report (--page raw) into a small JSON for profiles/.

python tools/ncu_summary.py REPORT.ncu-rep OUT.json [note]"""
import csv
import io
import json
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
           "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
           "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
           "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
           "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    note = sys.argv[3] if len(sys.argv) > 3 else ""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    kern = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        e = {"kernel": d["Kernel Name"].split("(")[0]}
        for m in METRICS:
            if m in d and d[m] != "":
                u = units[h.index(m)]
                try:
                    v = float(d[m].replace(",", ""))
                except ValueError:
                    v = d[m]
                e[m] = v
                if u:
                    e[m + ".unit"] = u
        kern.append(e)
    json.dump({"report": rep, "note": note, "kernels": kern}, open(out, "w"), indent=1)
    print(out, len(kern), "kernels")


if __name__ == "__main__":
    main()
