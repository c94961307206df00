# Per-launch figures of one `ncu --set full` capture, for profiles/r01_ncu.json:
#   python tools/ncu_summary.py REPORT.ncu-rep
import csv, io, json, subprocess, sys

KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "regs",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_active_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "launch__waves_per_multiprocessor": "waves",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
        "ns": 1, "us": 1e3, "ms": 1e6,
        "msecond": 1e6}


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, val = rows[0], rows[1], rows[2]
    res = {"kernel": val[hdr.index("Kernel Name")][:120]}
    for k, name in KEYS.items():
        if k in hdr:
            i = hdr.index(k)
            v = float(val[i].replace(",", ""))
            res[name] = v * UNIT.get(units[i], 1)
    res["duration_us"] = res.pop("duration_ns", 0.0) / 1e3
    res["dram_read_bytes"] = int(res.pop("dram_read", 0))
    res["dram_write_bytes"] = int(res.pop("dram_write", 0))
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
