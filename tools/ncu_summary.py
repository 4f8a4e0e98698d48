"""Summarise an `ncu --set full` raw-page CSV of tools/profile_set.py into the evidence files:

    python tools/ncu_summary.py RAW.csv[.gz] PSET.log OUT_PREFIX [--workload-map ebgan_b256_fp32=ebgan_l2:fp32,...]

profile_set.py warms every layer up, then runs each once after a unit_floats marker launch; the
launches between markers belong to the layer PSET.log lists at that position. Writes OUT_PREFIX.csv (one row per
kernel launch: layer, kernel, duration, DRAM bytes read / written, tensor-pipe / DRAM / L2 / issue
utilisation, registers) and merges per-layer DRAM traffic of each layer's main kernel into
profiles/ncu_traffic.json (bench.py reports it as roofline.traffic).
"""
import csv
import gzip
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
COLS = {"duration_ms": "gpu__time_duration.sum", "dram_read_gb": "dram__bytes_read.sum",
        "dram_write_gb": "dram__bytes_write.sum",
        "tensor_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l2_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "issue_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "regs": "launch__registers_per_thread"}
SCALE = {"ms": 1.0, "us": 1e-3, "ns": 1e-6, "Gbyte": 1.0, "Mbyte": 1e-3, "Kbyte": 1e-6, "byte": 1e-9}


def main():
    raw, pset, prefix = sys.argv[1:4]  # noqa: (usage in the docstring)
    opener = gzip.open if raw.endswith(".gz") else open
    rows = list(csv.reader(opener(raw, "rt")))
    head, units, data = rows[0], rows[1], rows[2:]
    idx = {k: head.index(v) for k, v in COLS.items()}
    kname = head.index("Kernel Name")
    labels = [ln.split(":")[0] + ":" + ln.split(":")[1] for ln in open(pset) if ":" in ln]
    # the measured pass: after the last len(labels) unit_floats markers, one group per layer
    marks = [i for i, r in enumerate(data) if "unit_floats" in r[kname]][-len(labels):]
    out, per_layer = [], {}
    for li, start in enumerate(marks):
        stop = marks[li + 1] if li + 1 < len(marks) else len(data)
        for r in data[start + 1:stop]:
            rec = {"layer": labels[li], "kernel": r[kname][:90]}
            for k, i in idx.items():
                v = float(r[i]) if r[i] not in ("", "n/a") else None
                if v is not None and k in ("duration_ms", "dram_read_gb", "dram_write_gb"):
                    v *= SCALE.get(units[i], 1.0)
                rec[k] = v
            out.append(rec)
            per_layer.setdefault(labels[li], []).append(rec)
    with open(prefix + ".csv", "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=list(out[0].keys()))
        w.writeheader()
        w.writerows(out)
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for lab, recs in per_layer.items():
        name, dtype = lab.split(":")
        wl = ("ebgan" if name.startswith("ebgan") else "dcgan" if name.startswith("dcgan") else
              "dataset" if name.startswith("ds") else "mnist")
        batch = {"ebgan": 256, "dcgan": 256, "dataset": 64, "mnist": 64}[wl]
        key = f"{wl}_b{batch}_{dtype}"
        traffic.setdefault(key, {})[name] = sum((r["dram_read_gb"] or 0) + (r["dram_write_gb"] or 0)
                                                for r in recs) * 1e9
    with open(tpath, "w") as f:
        json.dump(traffic, f, indent=1, sort_keys=True)
    for r in out:
        print(f"{r['layer']:<18} {r['kernel'][:44]:<44} {r['duration_ms']:.4f} ms  R {r['dram_read_gb']:.3f} "
              f"W {r['dram_write_gb']:.3f} GB  tensor {r['tensor_pct'] or 0:5.1f}%  dram {r['dram_pct'] or 0:5.1f}%")


if __name__ == "__main__":
    main()
