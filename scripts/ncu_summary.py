"""Summarise an ncu --set full report into profiles/*.json (run where ncu is
installed; reads the report with `ncu -i --page raw --csv`).

    python scripts/ncu_summary.py gpurun_out/prof_full.ncu-rep profiles/r01_ncu.json "c2 ..."
"""
import csv
import io
import json
import re
import subprocess
import sys

METRICS = {
    "duration_us": ("gpu__time_duration.sum", 1.0),
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "dram_throughput_pct": ("dram__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "l2_hit_rate_pct": ("lts__t_sector_hit_rate.pct", 1.0),
    "l2_throughput_pct": ("lts__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "fp64_pipe_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "ipc_per_sm": ("sm__inst_executed.avg.per_cycle_active", 1.0),
    "warps_active_per_sm": ("sm__warps_active.avg.per_cycle_active", 1.0),
    "registers_per_thread": ("launch__registers_per_thread", 1.0),
    "smem_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1.0),
    "smem_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1.0),
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
              "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,
              "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}


def main(rep, out, note):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    kernels = {}
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        name = re.sub(r"^void (<unnamed>::)?", "", d.get("Kernel Name", "?")).split("(")[0]
        short = name.split("<")[0]
        ent = {"kernel": name}
        for key, (m, _) in METRICS.items():
            if m not in d or d[m] in ("", "n/a"):
                continue
            v = float(d[m].replace(",", ""))
            if v != v:          # NaN (metric not collected for this launch)
                continue
            unit = u.get(m, "")
            if key.endswith("_bytes"):
                v *= UNIT_SCALE.get(unit, 1)
                v = int(round(v))
            elif key == "duration_us":
                v *= UNIT_SCALE.get(unit, 1)
            ent[key] = v
        # every pipe-utilisation counter the capture holds (tensor/DMMA, FMA, FP64, ALU, ...)
        pipes = {}
        for h, v in d.items():
            m = re.match(r"sm__pipe_(\w+?)_cycles_active\.avg\.pct_of_peak_sustained_active$", h)
            if m and v not in ("", "n/a"):
                try:
                    pipes[m.group(1)] = round(float(v.replace(",", "")), 2)
                except ValueError:
                    pass
            m = re.match(r"sm__inst_executed_pipe_(\w+?)\.avg\.pct_of_peak_sustained_active$", h)
            if m and v not in ("", "n/a"):
                try:
                    pipes["inst_" + m.group(1)] = round(float(v.replace(",", "")), 2)
                except ValueError:
                    pass
        if pipes:
            ent["pipes_pct_of_peak_active"] = dict(sorted(pipes.items(), key=lambda kv: -kv[1]))
        for key, m in (("issue_active_pct", "sm__issue_active.avg.pct_of_peak_sustained_active"),
                       ("l1tex_throughput_pct", "l1tex__throughput.avg.pct_of_peak_sustained_active"),
                       ("lts_bytes", "lts__t_bytes.sum"),
                       ("sm_throughput_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed")):
            if m in d and d[m] not in ("", "n/a"):
                try:
                    v = float(d[m].replace(",", ""))
                    if key == "lts_bytes":
                        v = int(v * UNIT_SCALE.get(u.get(m, ""), 1))
                    ent[key] = v
                except ValueError:
                    pass
        stalls = []
        for h, v in d.items():
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    stalls.append((float(v.replace(",", "")), h[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1.0
        stalls.sort(reverse=True)
        ent["top_stalls_pct"] = {h: round(100 * v / tot, 1) for v, h in stalls[:5]}
        kernels.setdefault(short, ent)
    with open(out, "w") as f:
        json.dump({"source": note, "kernels": kernels}, f, indent=1)
    print(json.dumps(kernels, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else rep)
