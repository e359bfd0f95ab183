"""Summarise an `ncu --set full` report into the JSON bench.py reads
(per-kernel duration, DRAM bytes per launch, throughput, occupancy, DMMA use).

python scripts/ncu_summary.py gpurun_out/prof_r01b.ncu-rep profiles/ncu_summary_r01.json "<source note>"
"""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": ("duration_us", 1e-3),
    "dram__bytes_read.sum": ("dram_read", 1.0),
    "dram__bytes_write.sum": ("dram_write", 1.0),
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": ("dram_throughput_pct", 1.0),
    "sm__warps_active.avg.pct_of_peak_sustained_active": ("warps_active_pct", 1.0),
    "launch__registers_per_thread": ("registers", 1.0),
    "launch__grid_size": ("grid", 1.0),
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active": ("dmma_inst_pct_of_peak_active", 1.0),
    "lts__t_sector_hit_rate.pct": ("l2_hit_pct", 1.0),
}
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1.0, "us": 1e3, "ms": 1e6, "usecond": 1e3,
        "nsecond": 1.0, "msecond": 1e6}


def main(rep, out, note):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    kernels = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").strip()
        rec = {}
        for m, (key, _) in METRICS.items():
            if m not in d or d[m] == "":
                continue
            v = float(d[m].replace(",", ""))
            u = units[hdr.index(m)]
            if key in ("dram_read", "dram_write"):
                v *= UNIT.get(u, 1.0)
            elif key == "duration_us":
                v = v * UNIT.get(u, 1.0) / 1e3
            rec[key] = v
        rec["dram_bytes_per_launch"] = rec.pop("dram_read", 0.0) + rec.pop("dram_write", 0.0)
        kernels.setdefault(name, []).append(rec)
    summary = {}
    for name, recs in kernels.items():
        keys = recs[0].keys()
        summary[name] = {k: round(sum(r[k] for r in recs) / len(recs), 3) for k in keys}
        summary[name]["launches_captured"] = len(recs)
    spmv = "k_bsr3_spmv_pcg" if "k_bsr3_spmv_pcg" in summary else "k_spmv_pcg"
    doc = {"source": note, "kernels": summary,
           "k_spmv_pcg": {"kernel": spmv, "dram_bytes_per_launch": summary.get(spmv, {}).get("dram_bytes_per_launch")}}
    with open(out, "w") as fh:
        json.dump(doc, fh, indent=1)
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else sys.argv[1])
