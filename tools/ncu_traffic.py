#!/usr/bin/env python
"""profiles/ncu_traffic.json from steady-state `ncu --set full` captures (launches taken after
--launch-skip, i.e. CG iterations with every column active): per workload and kernel class, the
median dram__bytes_read.sum + dram__bytes_write.sum per launch of the fp32 probe kernels.
Writes that are still dirty in the 126 MB L2 when a launch ends are not counted by ncu, so the
write share is a lower bound.  Under "<workload>_pipes": the median utilisation (% of peak,
sustained while active) of the pipes that bound each class -- DRAM, L1TEX (global + shared
memory traffic), the shared-memory wavefronts alone, instruction issue, the FMA pipe -- so a
kernel that is not HBM-bound shows what it is bound by.
    python tools/ncu_traffic.py C4=gpurun_out/v7_C4_full.ncu-rep C3=... C5=...
"""
import csv
import io
import json
import os
import statistics
import subprocess
import sys

CLASSES = [("k1k_rows_inv<float>", "dct_rows_inv"), ("k1k_cols<float>", "dct_cols"),
           ("k1k_rows_fwd<float>", "dct_rows_fwd"), ("k_update<float", "pcg_update"),
           ("k_conv_fft<float>", "conv_apply"), ("k_tc_phiP", "dense_phi_p"), ("k_tc_phiTW", "dense_phiT_w"),
           ("k_dir<float>", "pcg_direction")]


PIPES = {"dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
         "l1tex_pct": "l1tex__throughput.avg.pct_of_peak_sustained_active",
         "shared_wavefront_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
         "issue_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
         "fma_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"}


def pipes(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    kn = h.index("Kernel Name")
    per = {}
    for r in rows[2:]:
        for pat, cls in CLASSES:
            if pat in r[kn]:
                d = per.setdefault(cls, {})
                for key, metric in PIPES.items():
                    if metric in h and r[h.index(metric)]:
                        d.setdefault(key, []).append(float(r[h.index(metric)].replace(",", "")))
                break
    return {c: {k: round(statistics.median(v), 1) for k, v in d.items()} for c, d in per.items()}


def traffic(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    kn, rd, wr = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    units = rows[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    per = {}
    for r in rows[2:]:
        for pat, cls in CLASSES:
            if pat in r[kn]:
                b = float(r[rd]) * scale[units[rd]] + float(r[wr]) * scale[units[wr]]
                per.setdefault(cls, []).append(b)
                break
    return {c: int(statistics.median(v)) for c, v in per.items()}


if __name__ == "__main__":
    path = os.path.join(os.path.dirname(__file__), "..", "profiles", "ncu_traffic.json")
    doc = {"_doc": __doc__.strip().split("\n    python")[0].replace("\n", " ")}
    for arg in sys.argv[1:]:
        wl, rep = arg.split("=", 1)
        doc[wl] = traffic(rep)
        doc[wl + "_pipes"] = pipes(rep)
    json.dump(doc, open(path, "w"), indent=1)
    print(json.dumps(doc, indent=1))
