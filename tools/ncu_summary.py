"""Per-launch summaries of an `ncu --set full` capture exported with
`ncu -i X.ncu-rep --page raw --csv > X.csv`: one JSON object per launch (kernel,
duration, DRAM bytes, fp64 / tensor pipe activity, registers, occupancy, shared
wavefronts and bank conflicts), the numbers profiles/*.json carry.

    python tools/ncu_summary.py X.csv [name_regex]
"""
import csv
import json
import re
import sys

FIELDS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),
    "dram_read_GB": ("dram__bytes_read.sum", 1e-9),
    "dram_write_GB": ("dram__bytes_write.sum", 1e-9),
    "fp64_pipe_active_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed", 1.0),
    "fp64_inst_pct_of_active": ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", 1.0),
    "dmma_inst_pct_of_active": ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", 1.0),
    "tensor_pipe_active_pct": ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
                               1.0),
    "registers": ("launch__registers_per_thread", 1.0),
    "achieved_occupancy_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1.0),
    "shared_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1.0),
    "shared_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1.0),
}
# ncu reports bytes in the unit row (byte / Kbyte / Mbyte / Gbyte) and times in ns/us/ms
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1.0, "usecond": 1e3, "msecond": 1e6,
        "ns": 1.0, "us": 1e3, "ms": 1e6}


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
    head, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(head, r))
        u = dict(zip(head, units))
        name = d.get("Kernel Name", "")
        if pat and not pat.search(name):
            continue
        rec = {"kernel": re.sub(r"\(.*", "", name).replace("(anonymous namespace)::", "")}
        for k, (m, sc) in FIELDS.items():
            if m not in d:
                continue
            try:
                v = float(d[m].replace(",", ""))
            except ValueError:
                continue
            if "bytes" in m or "duration" in m:
                v *= UNIT.get(u.get(m, ""), 1.0)
            rec[k] = round(v * sc, 6)
        out.append(rec)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
