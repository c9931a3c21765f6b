"""profiles/ncu_traffic.json from the reports scripts/ncu_traffic.sh writes (gpurun_out/fwd_<config>.ncu-rep):
per workload and bench stage, the kernel's duration and DRAM bytes (cold, clean L2 per kernel)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

STAGE = (("k_front", "front"), ("k_aa_token", "fused_permute_aa"), ("k_aa_bulk", "fused_permute_aa"),
         ("k_unpermute", "unpermute_combine"))
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "usecond": 1.0,
         "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}
METRICS = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum")


def read(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], dict(zip(rows[0], rows[1]))
    res = {}
    for r in rows[2:]:
        d = dict(zip(head, r))
        name = d["Kernel Name"].replace("void ", "").split("(")[0]
        stage = next((s for key, s in STAGE if key in name), None)
        if stage is None or stage in res:
            continue
        v = {m: float(d[m].replace(",", "")) * SCALE[units[m]] for m in METRICS}
        res[stage] = {"kernel": name, "duration_us": v[METRICS[0]], "dram_read_bytes": v[METRICS[1]],
                      "dram_write_bytes": v[METRICS[2]], "traffic": v[METRICS[1]] + v[METRICS[2]]}
    return res


def main():
    src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out")
    wl = {}
    for name, (cfg, _topo) in bench.WORKLOADS.items():
        rep = os.path.join(src, f"fwd_{name}.ncu-rep")
        if os.path.exists(rep):
            wl[cfg["workload"]] = read(rep)
    doc = {"workloads": wl,
           "note": "ncu --set full --clock-control none (cache control all: cold, clean L2 per kernel) on "
                   "python bench.py --config <c> --quick at N=1 (scripts/ncu_traffic.sh); writes still resident "
                   "in L2 at kernel end are not counted (written back during the next kernel)"}
    with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main()
