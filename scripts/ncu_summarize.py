"""Summarise gpurun_out/ncu_<config>_<kernel>.csv (ncu --set full raw pages,
one launch each, from scripts/ncu_traffic.sh) into profiles/<round>_ncu_kernels.json:
per (config, kernel) duration, DRAM read/write bytes, L2 (lts) bytes, tensor-pipe
and throughput percentages.  bench.py reads it to fill roofline.traffic."""
import csv, glob, json, os, sys

ROUND = sys.argv[1] if len(sys.argv) > 1 else "r01"
KEYS = {
    "duration_us": ("gpu__time_duration.sum", 1e-3),  # ns -> us (ncu reports usecond or nsecond; handled below)
    "dram_read_bytes": ("dram__bytes_read.sum", 1),
    "dram_write_bytes": ("dram__bytes_write.sum", 1),
    "l2_bytes": ("lts__t_sectors.sum", 1),
    "tensor_pipe_pct_elapsed": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1),
    "tf32_tensor_ops_pct_of_peak": ("sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed", 1),
    "dram_throughput_pct": ("dram__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "l2_throughput_pct": ("lts__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "registers_per_thread": ("launch__registers_per_thread", 1),
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3,
        "ns": 1e-3, "us": 1, "ms": 1e3, "sector": 32,
        "%": 1, "register/thread": 1, "": 1}
out = {}
for path in sorted(glob.glob("gpurun_out/ncu_*.csv")):
    base = os.path.basename(path)[4:-4]
    if base.endswith("_details"):
        continue
    cfg, kern = base.split("_", 1)
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        continue
    h, units = rows[0], rows[1]
    # a bench kernel name can cover several launches (e.g. split-K GEMM + its
    # finish, CSC ranges + sparse dW): sizes and times add up over the distinct
    # kernel functions, percentages are duration-weighted; repeated launches of
    # the same function (the range of another step) are averaged
    by_fn = {}
    for r in rows[2:]:
        by_fn.setdefault(r[h.index("Kernel Name")], []).append(r)
    launches = [v[0] for v in by_fn.values()]
    reps = [len(v) for v in by_fn.values()]
    d = {"kernel_function": " + ".join(r[h.index("Kernel Name")][:80] for r in launches),
         "grid": " + ".join(r[h.index("Grid Size")] for r in launches), "launches": len(launches),
         "captured_per_function": reps}
    vals = []
    for group in by_fn.values():
        one, cnt = {}, {}
        for r in group:
            for k, (m, _) in KEYS.items():
                if m in h:
                    i = h.index(m)
                    try:
                        one[k] = one.get(k, 0.0) + float(r[i].replace(",", "")) * UNIT.get(units[i], 1)
                        cnt[k] = cnt.get(k, 0) + 1
                    except ValueError:
                        pass
        vals.append({k: v / cnt[k] for k, v in one.items()})
    tot_t = sum(v.get("duration_us", 0) for v in vals) or 1.0
    for k in KEYS:
        if not any(k in v for v in vals):
            continue
        if k.endswith("_pct") or "pct" in k:
            d[k] = sum(v.get(k, 0) * v.get("duration_us", 0) for v in vals) / tot_t
        elif k == "registers_per_thread":
            d[k] = max(v.get(k, 0) for v in vals)
        else:
            d[k] = sum(v.get(k, 0) for v in vals)
    if "dram_read_bytes" in d and "dram_write_bytes" in d:
        d["dram_bytes"] = d["dram_read_bytes"] + d["dram_write_bytes"]
    if "duration_us" in d:
        if "dram_bytes" in d:
            d["dram_gbs"] = d["dram_bytes"] / d["duration_us"] / 1e3
        if "l2_bytes" in d:
            d["l2_gbs"] = d["l2_bytes"] / d["duration_us"] / 1e3
    out.setdefault(cfg, {})[kern] = d
meta = {"how": "ncu --set full --clock-control none, one launch per (config, kernel) selected by the library's "
               "NVTX range (HB_NVTX=1, eager step); cold caches between ncu replay passes, so durations are "
               "serialized cold-cache times (shares, not absolutes); scripts/ncu_traffic.sh + scripts/ncu_summarize.py"}
json.dump({"meta": meta, "kernels": out}, open(f"profiles/{ROUND}_ncu_kernels.json", "w"), indent=1)
for cfg, ks in out.items():
    for k, d in ks.items():
        print(f"{cfg:9s} {k:22s} {d.get('duration_us', 0):8.1f} us  dram {d.get('dram_bytes', 0)/1e6:8.1f} MB "
              f"({d.get('dram_gbs', 0):6.0f} GB/s)  L2 {d.get('l2_bytes', 0)/1e6:8.1f} MB ({d.get('l2_gbs', 0):6.0f} GB/s)"
              f"  tensor {d.get('tensor_pipe_pct_elapsed', 0):5.1f}%  l2thr {d.get('l2_throughput_pct', 0):5.1f}%")
