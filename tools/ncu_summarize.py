"""Summarise ncu --set full reports (read here with `ncu -i`): per launch kernel name, duration,
DRAM bytes, achieved DRAM bandwidth, tensor-pipe and SM throughput.
Usage: python tools/ncu_summarize.py gpurun_out/prof_attn.ncu-rep [...]"""
import csv, io, subprocess, sys

WANT = {
    "gpu__time_duration.sum": "time",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm%",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem%",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tmem/umma%",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed": "hmma%",
    "launch__grid_size": "grid",
    "launch__registers_per_thread": "regs",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ%",
    "lts__t_sector_hit_rate.pct": "l2hit%",
}


def unit_scale(u):
    return {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "byte": 1,
            "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "Tbyte": 1e12,
            "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1.0)


for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        print(rep, "no data"); continue
    hdr, units = rows[0], rows[1]
    idx = {k: hdr.index(k) for k in WANT if k in hdr}
    name_i = hdr.index("Kernel Name")
    print(f"== {rep}")
    for r in rows[2:]:
        v = {}
        for k, i in idx.items():
            try:
                v[WANT[k]] = float(r[i].replace(",", "")) * unit_scale(units[i])
            except ValueError:
                v[WANT[k]] = float("nan")
        t = v.get("time", float("nan"))
        rd, wr = v.get("dram_rd", 0), v.get("dram_wr", 0)
        print(f"{r[name_i][:60]:60s} {t*1e6:8.1f} us  dram {rd/1e6:9.1f}+{wr/1e6:7.1f} MB "
              f"{(rd+wr)/t/1e9 if t else 0:7.0f} GB/s  " +
              "  ".join(f"{k} {v[k]:.0f}" for k in ("sm%", "mem%", "tmem/umma%", "hmma%", "occ%", "l2hit%", "grid", "regs") if k in v))
