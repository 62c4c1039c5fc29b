"""Summarise an ncu report (run HERE, no GPU): per-kernel duration, DRAM bytes, pipe and
issue utilisation; optionally write profiles/ncu_traffic.json for bench.py's roofline."""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__cycles_elapsed.avg", "sm__cycles_active.avg", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.per_cycle_active",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def main(rep, out_json=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        ent = {"kernel": d.get("Kernel Name", "")[:60], "grid": d.get("launch__grid_size"),
               "block": d.get("launch__block_size")}
        for k in KEYS:
            if k in d:
                ent[k] = f"{d[k]} {u.get(k, '')}".strip()
        res.append(ent)
    for e in res:
        print(json.dumps(e))
    if out_json:
        def to_bytes(s):
            v, unit = s.split()[0], s.split()[1] if len(s.split()) > 1 else "byte"
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            return float(v.replace(",", "")) * mult
        per = [to_bytes(e["dram__bytes_read.sum"]) + to_bytes(e["dram__bytes_write.sum"])
               for e in res if "wl_gemv" in e["kernel"]]
        # mean over the captured launches (one decoder layer: qkv, o, gate/up, down), the
        # same averaging as bench.py's per-launch roofline
        json.dump({"source": rep, "dram_bytes_per_launch": sum(per) / len(per) if per else None,
                   "per_launch": per, "kernels": res}, open(out_json, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
