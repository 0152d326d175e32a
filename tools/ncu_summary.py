"""Summarise ncu --set full captures (one kernel launch each) into JSON:
python tools/ncu_summary.py <tag>=<file.ncu-rep> ...  -> prints {tag: {...}}"""
import csv, io, json, subprocess, sys

KEYS = {"gpu__time_duration.sum": "duration_ms", "dram__bytes_read.sum": "dram_bytes_read",
        "dram__bytes_write.sum": "dram_bytes_write", "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
        "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1tex_throughput_pct",
        "launch__registers_per_thread": "registers", "launch__grid_size": "grid", "launch__block_size": "block",
        "sm__cycles_elapsed.avg.per_second": "sm_clock_ghz"}
SCALE = {"ms": 1.0, "us": 1e-3, "ns": 1e-6, "s": 1e3, "msecond": 1.0, "usecond": 1e-3, "nsecond": 1e-6,
         "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12, "GHz": 1e9, "MHz": 1e6,
         "cycle/second": 1.0, "cycle/nsecond": 1e9, "cycle/usecond": 1e6}


def summary(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else None}
    for k, name in KEYS.items():
        if k in hdr:
            i = hdr.index(k)
            try:
                v = float(vals[i].replace(",", ""))
            except ValueError:
                continue
            u = units[i]
            if name == "duration_ms":
                v *= SCALE.get(u, 1.0)
            elif u in SCALE:
                v *= SCALE[u]
            out[name] = v
    for i, k in enumerate(hdr):   # tensor-pipe and TMEM counters, whatever this ncu names them
        if ("tensor" in k or "tmem" in k) and "pct" in k:
            try:
                out[k] = float(vals[i].replace(",", ""))
            except ValueError:
                pass
    if "dram_bytes_read" in out and "duration_ms" in out:
        out["dram_tbs"] = (out["dram_bytes_read"] + out.get("dram_bytes_write", 0.0)) / (out["duration_ms"] * 1e-3) / 1e12
    return out


if __name__ == "__main__":
    res = {}
    for a in sys.argv[1:]:
        tag, path = a.split("=", 1)
        res[tag] = summary(path)
    print(json.dumps(res, indent=1))
