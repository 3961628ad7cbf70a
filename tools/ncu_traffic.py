"""Extract per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of each kernel from an
`ncu --set full` report into profiles/<tag>_traffic.json, which bench.py reads for roofline.traffic.

    python tools/ncu_traffic.py gpurun_out/x.ncu-rep cfg3 profiles/r2_traffic.json
"""
import csv
import io
import json
import os
import subprocess
import sys


def main():
    rep, workload, out = sys.argv[1], sys.argv[2], sys.argv[3]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    data = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].split("<")[0].split("::")[-1].replace("_kernel", "")

        def f(k):
            return float(d.get(k, "0").replace(",", "") or 0)
        b = f("dram__bytes_read.sum") + f("dram__bytes_write.sum")
        unit = d.get("dram__bytes_read.sum", "")
        data.setdefault(name, []).append(b)
    units = dict(zip(hdr, rows[1]))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units.get("dram__bytes_read.sum", "byte"), 1)
    res = json.load(open(out)) if os.path.exists(out) else {}
    res.setdefault(workload, {})
    for k, v in data.items():
        res[workload][k] = max(v) * scale
    res["_source"] = f"ncu --set full report {os.path.basename(rep)}: dram__bytes_read.sum + dram__bytes_write.sum, max over launches"
    json.dump(res, open(out, "w"), indent=1, sort_keys=True)
    print(json.dumps(res[workload], indent=1))


if __name__ == "__main__":
    main()
