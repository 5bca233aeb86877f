"""Summarise gpurun_out/prof_*.ncu-rep + launches_decode.csv into profiles/.
Algorithmic bytes per launch: decode weights/KV as in tenants.DecodeModel
(one layer), GEMM operands 3 x 8192^2 x 2 B."""
import csv, io, json, os, subprocess, sys, collections

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles")
TAG = sys.argv[1] if len(sys.argv) > 1 else "r1"
ALG = {"attn": 2 * 32 * 8 * 1024 * 128 * 2, "gate_up": 2 * 14336 * 4096 * 2, "lm_head": 128256 * 4096 * 2,
       "qkv": 6144 * 4096 * 2, "o": 4096 * 4096 * 2, "down": 4096 * 14336 * 2, "gemm": 3 * 8192 * 8192 * 2}
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sectors.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum"]
SCALE = {"ms": 1e-3, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "nsecond": 1e-9, "s": 1.0, "second": 1.0,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
summary = {"round": TAG, "source": "ncu --set full --clock-control none --import-source on -k regex:ds_solo_kernel -s 1 -c 1 "
           "(solo plain-grid launch of the same body; the persistent executor cannot be replayed by ncu)",
           "kernels": {}}
for k, alg in ALG.items():
    rep = os.path.join(ROOT, "gpurun_out", f"prof_{k}.ncu-rep")
    if not os.path.exists(rep):
        continue
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    with open(os.path.join(OUT, f"{TAG}_ncu_raw_{k}.csv"), "w") as f:
        w = csv.writer(f)
        idx = [i for i, h in enumerate(hdr) if any(h.startswith(p) for p in ("gpu__", "dram__", "sm__", "lts__", "l1tex__", "launch__", "smsp__inst"))]
        w.writerow([hdr[i] for i in idx]); w.writerow([units[i] for i in idx]); w.writerow([vals[i] for i in idx])
    d = {}
    for key in KEYS:
        if key in hdr:
            i = hdr.index(key)
            try:
                d[key] = {"value": float(vals[i].replace(",", "")), "unit": units[i]}
            except ValueError:
                pass
    dur = d["gpu__time_duration.sum"]["value"] * SCALE.get(d["gpu__time_duration.sum"]["unit"], 1)
    rd = d["dram__bytes_read.sum"]["value"] * SCALE.get(d["dram__bytes_read.sum"]["unit"], 1)
    wr = d["dram__bytes_write.sum"]["value"] * SCALE.get(d["dram__bytes_write.sum"]["unit"], 1)
    d["traffic_bytes"] = rd + wr
    d["algorithmic_bytes"] = alg
    d["traffic_over_algorithmic"] = round((rd + wr) / alg, 3)
    d["duration_s"] = dur
    d["achieved_GBps_algorithmic"] = round(alg / dur / 1e9, 1)
    summary["kernels"][k] = d
# launch list: share of one decode step per kernel body (solo, serialised, cold)
lpath = os.path.join(ROOT, "gpurun_out", "launches_decode.csv")
if os.path.exists(lpath):
    lines = [l for l in open(lpath) if not l.startswith("==")]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    rows = [r for r in rows if r.get("Metric Name") == "gpu__time_duration.sum"]
    solo = [r for r in rows if "ds_solo_kernel" in r["Kernel Name"]]
    with open(os.path.join(OUT, f"{TAG}_launches_decode_step.csv"), "w") as f:
        f.write("launch,kernel,gpu__time_duration_ns\n")
        for r in rows:
            v = float(r["Metric Value"].replace(",", ""))
            unit = r.get("Metric Unit", "ns")
            ns = v * {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1)
            f.write(f'{r["ID"]},{r["Kernel Name"][:80].replace(",", ";")},{int(ns)}\n')
    summary["launch_list"] = {"file": f"{TAG}_launches_decode_step.csv", "solo_body_launches": len(solo)}
    # label the solo launches by decode-step order (profile_solo.py decode: 2 steps of
    # embed, 32 x (qkv, attn, o, gate_up, down), lm_head, argmax) and average per kernel:
    # the serialised cold-cache counterpart of the bench's per-kernel CUDA-event times
    order = ["embed"] + ["qkv", "attn", "o", "gate_up", "down"] * 32 + ["lm_head", "argmax"]
    def ns_of(r):
        v = float(r["Metric Value"].replace(",", ""))
        return v * {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(r.get("Metric Unit", "ns"), 1)
    if len(solo) % len(order) == 0:
        per = collections.defaultdict(list)
        for i, r in enumerate(solo):
            per[order[i % len(order)]].append(ns_of(r))
        step_ns = sum(ns_of(r) for r in solo) / (len(solo) // len(order))
        byts = {"qkv": 6144 * 4096 * 2, "attn": 2 * 32 * 8 * 1024 * 128 * 2, "o": 4096 * 4096 * 2,
                "gate_up": 2 * 14336 * 4096 * 2, "down": 4096 * 14336 * 2, "lm_head": 128256 * 4096 * 2}
        hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
            os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6553.6
        summary["launch_list"]["per_kernel_us"] = {
            k: {"mean_us": round(sum(v) / len(v) / 1e3, 2), "launches_per_step": len(v) * len(order) // len(solo),
                "share_of_step": round(sum(v) / (len(solo) // len(order)) / step_ns, 4),
                **({"hbm_frac": round(byts[k] / (sum(v) / len(v)) / hbm, 4)} if k in byts else {})}
            for k, v in per.items()}
        summary["launch_list"]["step_ms_serialised"] = round(step_ns / 1e6, 4)
json.dump(summary, open(os.path.join(OUT, f"{TAG}_ncu_summary.json"), "w"), indent=1)
for k, d in summary["kernels"].items():
    print(k, round(d["duration_s"] * 1e6, 1), "us", d["achieved_GBps_algorithmic"], "GB/s alg", "traffic/alg",
          d["traffic_over_algorithmic"], "tensor%", d.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", {}).get("value"))
