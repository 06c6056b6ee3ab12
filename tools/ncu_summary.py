"""Summarise an `ncu --set full` capture of the ring kernel into
profiles/ncu_engine_summary.json (bench.py reads `dram_bytes_per_launch`
from it for roofline.traffic) and a launch list into profiles/<round>/."""
import csv, json, subprocess, sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
rep, launches, rnd = sys.argv[1], sys.argv[2], sys.argv[3]
# optional: a batched capture -> profiles/<round>/ncu_c3_summary.json (argv[4] = "c3")
kind = sys.argv[4] if len(sys.argv) > 4 else "c2"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
r = list(csv.reader(raw))
h, u, v = r[0], r[1], r[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum.per_second",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
        "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
        "sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "lts__t_sector_hit_rate.pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]
out = {n: (v[i], u[i]) for i, n in enumerate(h) if n in want}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
num = lambda s: float(s.replace(",", ""))
t = num(out["gpu__time_duration.sum"][0]) * (1e3 if out["gpu__time_duration.sum"][1] == "ms" else 1)
rd = num(out["dram__bytes_read.sum"][0]) * scale[out["dram__bytes_read.sum"][1]]
wr = num(out["dram__bytes_write.sum"][0]) * scale[out["dram__bytes_write.sum"][1]]
alg = 15546859520 if kind == "c2" else 34780356608
summ = {"kernel": "vdc_dev::ring::ring_kernel" + ("" if kind == "c2" else "<true> (batched)"), "round": rnd,
        "capture": "ncu --set full --clock-control none --import-source on -k regex:ring_kernel -s 3 -c 1, " +
                   ("python bench.py --steps 1 --warmup 3 (32-layer Llama-3-8B decode, ctx 4096)" if kind == "c2" else
                    "python bench.py --batch 32 --steps 1 --warmup 3 (C3: 32-layer Llama-3-8B, batch 32, paged KV)"),
        "gpu_time_us": t, "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
        "algorithmic_bytes_per_launch": alg, "traffic_over_algorithmic": (rd + wr) / alg,
        "dram_gbps": (rd + wr) / t / 1e3, "metrics": {k: out[k][0] + " " + out[k][1] for k in out}}
if kind != "c2":
    (ROOT / "profiles" / rnd / f"ncu_{kind}_summary.json").write_text(json.dumps(summ, indent=1))
    print(json.dumps({k: summ[k] for k in ("gpu_time_us", "dram_bytes_per_launch", "traffic_over_algorithmic", "dram_gbps")}))
    sys.exit(0)
(ROOT / "profiles" / "ncu_engine_summary.json").write_text(json.dumps(summ, indent=1))
rows = list(csv.reader(open(launches)))
hdr = None
lines = ["# ncu --metrics gpu__time_duration.sum --clock-control none, python bench.py --steps 3 --warmup 3 --no-cpu-baseline",
         "# (cold-cache, serialised: compare shares, not absolutes). Non-ring launches are the device input synthesis (synth_kernel).",
         "# id | kernel | grid | block | gpu_time_ns"]
for row in rows:
    if row and row[0] == "ID":
        hdr = row
        continue
    if hdr and len(row) == len(hdr):
        d = dict(zip(hdr, row))
        lines.append(" | ".join([d["ID"], d["Kernel Name"].split("(")[0][:60], d["Grid Size"], d["Block Size"], d["Metric Value"]]))
(ROOT / "profiles" / rnd / "launches_bench.txt").write_text("\n".join(lines) + "\n")
print(json.dumps({k: summ[k] for k in ("gpu_time_us", "dram_bytes_per_launch", "traffic_over_algorithmic", "dram_gbps")}))
for k, (val, unit) in out.items():
    print(k, val, unit)
