"""Copy an r2_round.sh run (gpurun_out/) into tracked profiles/ (prefix TAG):
bench lines (all configs, reference arm, per-point API), launch lists, ncu
--set full summaries of the projection kernel (cfg 5 / cfg 2 launches) and the
stream kernel, their per-line warp-stall summaries, and profiles/traffic.json
(DRAM bytes per launch, read by bench.py for roofline.traffic).

    python scripts/save_r2.py TAG
"""
import csv
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"
tag = sys.argv[1]


def lines(src):
    return [l for l in (OUT / src).read_text().splitlines() if l.startswith("{")]


for src, dst in (("bench.json", "bench_all_configs.jsonl"), ("bench_ref.json", "bench_reference_all_configs.jsonl"),
                 ("bench_point.json", "bench_point_api.jsonl")):
    if (OUT / src).exists():
        (PROF / f"{tag}_{dst}").write_text("\n".join(lines(src)) + "\n")
for t in ("r5", "r2"):
    for ext in ("csv", "txt"):
        p = OUT / f"launches_{t}.{ext}"
        if p.exists():
            (PROF / f"{tag}_launches_cfg{t[1]}{'_summary' if ext == 'txt' else ''}.{ext}").write_text(p.read_text())

KEEP = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_op_red.sum", "lts__t_sectors_op_atom.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second"]
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
tr_path = PROF / "traffic.json"
traffic = {}  # rebuilt from this round's captures
for rep, cfg, name in (("prof_h5", 5, "ncu_hash_cfg5"), ("prof_h2", 2, "ncu_hash_cfg2"), ("prof_pair", 5, "ncu_stream_cfg5")):
    path = OUT / f"{rep}.ncu-rep"
    if not path.exists():
        continue
    raw = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    idx = [hdr.index(k) for k in KEEP if k in hdr]
    with open(PROF / f"{tag}_{name}_summary.csv", "w", newline="") as f:
        w = csv.writer(f)
        w.writerow([hdr[i] for i in idx])
        w.writerow([units[i] for i in idx])
        for r in rows[2:]:
            w.writerow([r[i] for i in idx])
    ir, iw, ik = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum"), hdr.index("Kernel Name")
    per = traffic.setdefault(f"cfg{cfg}", {})
    for r in rows[2:]:
        k = r[ik].split("(")[0].split("::")[-1].split("<")[0].strip()
        per[k] = float(r[ir]) * SCALE[units[ir]] + float(r[iw]) * SCALE[units[iw]]
    st = subprocess.run([sys.executable, str(ROOT / "scripts" / "ncu_lines.py"), str(path)], capture_output=True,
                        text=True).stdout
    (PROF / f"{tag}_{name}_stall_lines.txt").write_text("\n".join(st.splitlines()[:40]) + "\n")
traffic["source"] = (f"profiles/{tag}_ncu_hash_cfg5_summary.csv, {tag}_ncu_hash_cfg2_summary.csv, "
                     f"{tag}_ncu_stream_cfg5_summary.csv (ncu --set full, DRAM bytes per launch; the cfg 5 hashing "
                     "launch is one bench hashing group)")
tr_path.write_text(json.dumps(traffic, indent=1) + "\n")
print(json.dumps(traffic, indent=1))
