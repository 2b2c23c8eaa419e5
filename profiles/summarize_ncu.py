"""Summarise an ncu --set full capture (run here, no GPU needed):
    python profiles/summarize_ncu.py gpurun_out/prof.ncu-rep > profiles/<name>.txt"""
import csv
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "lts__t_sector_hit_rate.pct", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
    "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "nvlrx__bytes.sum", "nvltx__bytes.sum",
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"kernel: {name}")
        for k in KEYS:
            for i, h in enumerate(hdr):
                if h == k or h.endswith("." + k) or (k in h and h.startswith("TPC.") and k.startswith("TPC.")):
                    print(f"  {h} [{units[i]}] = {vals[i]}")
                    break
        try:
            rd = float(vals[hdr.index("dram__bytes_read.sum")])
            wr = float(vals[hdr.index("dram__bytes_write.sum")])
            ur = units[hdr.index("dram__bytes_read.sum")]
            uw = units[hdr.index("dram__bytes_write.sum")]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            print(f"  traffic_bytes (read+write) = {rd * scale.get(ur, 1) + wr * scale.get(uw, 1):.4e}")
        except ValueError:
            pass


if __name__ == "__main__":
    main(sys.argv[1])
