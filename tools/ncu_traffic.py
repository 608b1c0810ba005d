"""profiles/kernel_traffic.json from an `ncu --set full` report of the bench:
dram bytes (read + write) and duration per launch of each hot kernel.

    python tools/ncu_traffic.py REPORT.ncu-rep > profiles/kernel_traffic.json
"""
import csv
import io
import json
import subprocess
import sys

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}
HOT = ("mt_tc_kernel", "register_edges_kernel", "vh_insert_frames_kernel")
METRICS = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active")


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        kn = d["Kernel Name"]
        kn = kn[5:] if kn.startswith("void ") else kn  # templated kernels: "void name<...>(...)"
        name = next((h for h in HOT if kn.startswith(h)), None)
        if name is None or name in res:
            continue
        u = dict(zip(hdr, units))
        val = {m: float(d[m]) * UNIT.get(u[m], 1.0) if u[m] in UNIT else float(d[m]) for m in METRICS}
        res[name] = {"dram_bytes_per_launch": val["dram__bytes_read.sum"] + val["dram__bytes_write.sum"],
                     "dram_read_bytes": val["dram__bytes_read.sum"], "dram_write_bytes": val["dram__bytes_write.sum"],
                     "ncu_ms_per_launch": val["gpu__time_duration.sum"],
                     "tensor_pipe_active_pct": val[METRICS[3]], "alu_pipe_active_pct": val[METRICS[4]],
                     "issue_active_pct": val[METRICS[5]]}
    json.dump({"source": rep.split("/")[-1], "note": "one launch each, --clock-control none, cold cache",
               "kernels": res}, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1])
