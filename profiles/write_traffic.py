"""Record the DRAM traffic of ONE K6 launch (the bench's dominant kernel,
k_lsqr_pipe) from an `ncu --set full` capture into
profiles/lsqr_pass_traffic.json, stamped with the hash of the kernel's
source files so bench.py uses it only while the source is unchanged.

    python profiles/write_traffic.py <report.ncu-rep> <capture name> [n m]
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    rep, name = sys.argv[1], sys.argv[2]
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 24
    m = int(sys.argv[4]) if len(sys.argv) > 4 else 200
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    data = [dict(zip(hdr, r)) for r in rows[2:]]     # row 1 holds the units
    k6 = [d for d in data if "k_lsqr_pipe" in d.get("Kernel Name", "")]
    assert k6, "no k_lsqr_pipe launch in the report"
    d = k6[0]

    def val(key):
        return float(d[key].replace(",", ""))
    rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    dur = val("gpu__time_duration.sum")
    # the capture reports bytes unscaled only with --print-units base; the
    # raw page's second row gives the unit
    units = dict(zip(hdr, rows[1]))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd *= scale.get(units["dram__bytes_read.sum"], 1.0)
    wr *= scale.get(units["dram__bytes_write.sum"], 1.0)
    tscale = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}
    dur *= tscale.get(units["gpu__time_duration.sum"], 1.0)
    import bench
    rec = {"capture": name, "kernel": d["Kernel Name"][:120], "n": n, "m": m,
           "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
           "duration_s": dur, "algorithmic_bytes": 8.0 * n * (m + 2),
           "src_files": list(bench.TRAFFIC_SRC), "src_sha": bench.src_sha(bench.TRAFFIC_SRC)}
    json.dump(rec, open(os.path.join(ROOT, "profiles", "lsqr_pass_traffic.json"), "w"), indent=1)
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
