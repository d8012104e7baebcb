"""profiles/r2_attn_*_ncu.json from an `ncu --set full --profile-from-start off`
capture of bench.py's profiled attention launch and the bench's own JSON line
(same command): DRAM traffic and duration of that launch next to its
algorithmic bytes and context.

    python scripts/ncu_attn_json.py REPORT.ncu-rep BENCH_LINE.json OUT.json
"""
import csv
import io
import json
import subprocess
import sys


def main(rep, bench_json, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, r = rows[0], rows[1], rows[2]

    def val(name):
        i = hdr.index(name)
        v = float(r[i].replace(",", ""))
        u = units[i]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3,
                 "usecond": 1, "msecond": 1e3}.get(u, 1)
        return v * scale
    line = json.loads([ln for ln in open(bench_json) if ln.startswith("{")][-1])
    roof = line["roofline"]
    rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    dur = val("gpu__time_duration.sum")
    doc = {"kernel": r[hdr.index("Kernel Name")][:80],
           "source": f"ncu --set full --clock-control none --profile-from-start off -k "
                     f"regex:attn_mma -c 1 on bench.py ({rep})",
           "context": roof.get("context"), "algorithmic_bytes": roof["bytes_per_launch"],
           "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes": rd + wr,
           "traffic_over_algorithmic": round((rd + wr) / roof["bytes_per_launch"], 4),
           "duration_us": round(dur, 2),
           "dram_gbs_under_ncu": round((rd + wr) / dur / 1e3, 1),
           "algorithmic_gbs_under_ncu": round(roof["bytes_per_launch"] / dur / 1e3, 1),
           "bench_avg_launch_us": round(roof["avg_launch_ms"] * 1e3, 2),
           "dram_throughput_pct_of_peak": val("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
           "warps_active_pct": val("sm__warps_active.avg.pct_of_peak_sustained_active"),
           "registers_per_thread": val("launch__registers_per_thread"),
           "grid_size": val("launch__grid_size")}
    with open(out, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:4])
