"""Copy a round_check.sh run (gpurun_out/) into tracked profiles/ summaries.

    python scripts/save_profiles.py TAG [CFG]

writes profiles/TAG_bench_cfgN.json, TAG_bench_ref_cfgN.json,
TAG_launches_cfgN.csv / _summary.txt, TAG_ncu_full_cfgN_summary.csv and
updates profiles/traffic.json (DRAM bytes per launch of each profiled kernel,
read by bench.py for the roofline's `traffic`).
"""
import csv
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"
tag = sys.argv[1]
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 2

for src, dst in (("bench.json", f"{tag}_bench_cfg{cfg}.json"), ("bench_ref.json", f"{tag}_bench_ref_cfg{cfg}.json"),
                 ("launches.csv", f"{tag}_launches_cfg{cfg}.csv"),
                 ("launches.txt", f"{tag}_launches_cfg{cfg}_summary.txt")):
    if (OUT / src).exists():
        text = (OUT / src).read_text()
        if src.endswith(".json"):
            text = text.strip().splitlines()[-1] + "\n"
        (PROF / dst).write_text(text)

rep = OUT / "prof_full.ncu-rep"
if rep.exists():
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    keep = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"]
    idx = [hdr.index(k) for k in keep if k in hdr]
    with open(PROF / f"{tag}_ncu_full_cfg{cfg}_summary.csv", "w", newline="") as f:
        w = csv.writer(f)
        w.writerow([hdr[i] for i in idx])
        w.writerow([units[i] for i in idx])
        for r in rows[2:]:
            w.writerow([r[i] for i in idx])
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tr_path = PROF / "traffic.json"
    traffic = json.loads(tr_path.read_text()) if tr_path.exists() else {}
    per = {}
    ir, iw, ik = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum"), hdr.index("Kernel Name")
    for r in rows[2:]:
        name = r[ik].split("(")[0].split("::")[-1].split("<")[0].strip()
        per[name] = float(r[ir]) * scale[units[ir]] + float(r[iw]) * scale[units[iw]]
    traffic[f"cfg{cfg}"] = per
    traffic["source"] = f"profiles/{tag}_ncu_full_cfg{cfg}_summary.csv (ncu --set full, DRAM bytes per launch)"
    tr_path.write_text(json.dumps(traffic, indent=1) + "\n")
    print(json.dumps(per, indent=1))
