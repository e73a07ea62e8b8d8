#!/usr/bin/env python3
"""profiles/ncu_step_kernel.json from an `ncu --set full` raw CSV of the bench's step kernel
(the `traffic` and `ncu` keys of bench.py's roofline object).

    python tools/ncu_json.py gpurun_out/r2/r2_step_r20_raw.csv "<kernel description>" "<source note>"
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(path, kernel, source):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    row = next(r for r in rows[2:] if "step_packed_ws3" in r[hdr.index("Kernel Name")])

    def val(name, scale_to=None):
        i = hdr.index(name)
        v = float(row[i])
        u = units[i]
        if scale_to == "B":
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
        if scale_to == "ms":
            v *= {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "msecond": 1.0, "usecond": 1e-3}[u]
        return v

    rd, wr = val("dram__bytes_read.sum", "B"), val("dram__bytes_write.sum", "B")
    dur = val("gpu__time_duration.sum", "ms")
    out = {
        "kernel": kernel,
        "source": source,
        "dram_bytes_read": int(rd),
        "dram_bytes_write": int(wr),
        "dram_bytes_per_launch": int(rd + wr),
        "algorithmic_bytes_per_launch": 871696100,
        "algorithmic_model": "packed: 3^20 cells x 2 bits (read own + write next state) = 871.7 MB; writes "
                             "below the model are dirty lines still in L2 when the launch ends",
        "ncu_duration_ms": dur,
        "dram_throughput_pct_of_peak": round(val("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"), 2),
        "dram_gbs": round((rd + wr) / (dur * 1e-3) / 1e9),
        "issue_slots_busy_pct": round(val("sm__inst_issued.avg.pct_of_peak_sustained_active"), 1),
        "achieved_warps_per_sm": round(val("sm__warps_active.avg.per_cycle_active"), 2),
        "registers_per_thread": int(val("launch__registers_per_thread")),
        "smem_per_cta_kb": round(val("launch__shared_mem_per_block_dynamic"), 2),
    }
    with open(os.path.join(ROOT, "profiles", "ncu_step_kernel.json"), "w") as fh:
        json.dump(out, fh, indent=2)
        fh.write("\n")
    print(json.dumps(out))


if __name__ == "__main__":
    main(*sys.argv[1:4])
