"""Writes profiles/ncu_traffic.json: DRAM bytes (read + write) per launch of
each workload's dominant kernel from one ncu capture, stamped with the content
hash of the library build it was measured on (libds2ctc.so.sha256), which
bench.py checks before reporting it as roofline.traffic. Run on the GPU box:

    python tools/ncu/traffic.py english:k_pair mandarin:k_dense_t
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
OUT = os.path.join(ROOT, "profiles", "ncu_traffic.json")
LIB = os.path.join(ROOT, "paper_1512_02595_b200", "libds2ctc.so")


def capture(workload: str, kernel: str):
    log = os.path.join(ROOT, "gpurun_out", f"traffic_{workload}.csv")
    os.makedirs(os.path.dirname(log), exist_ok=True)
    cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none", "-k", f"regex:{kernel}", "-c", "3", "--csv", "--log-file", log,
           sys.executable, os.path.join(ROOT, "bench.py"), "--workload", workload, "--steps", "1", "--warmup", "3",
           "--no-cpu-baseline", "--soak-seconds", "0"]
    subprocess.run(cmd, cwd=ROOT, stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL, timeout=900,
                   env=dict(os.environ, DS2CTC_HOST_CHUNKS="1"))
    rows = [r for r in csv.reader(open(log)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = {}
    for r in rows[1:]:
        if kernel.split("|")[0] not in r[ki]:
            continue
        per.setdefault(r[ii], {})[r[mi]] = float(r[vi].replace(",", ""))
    last = per[sorted(per, key=int)[-1]]  # the last launch: warm process, same inputs as the timed steps
    return {"bytes": last["dram__bytes_read.sum"] + last["dram__bytes_write.sum"],
            "read": last["dram__bytes_read.sum"], "write": last["dram__bytes_write.sum"],
            "ns": last["gpu__time_duration.sum"], "launches_seen": len(per)}


def main():
    with open(LIB + ".sha256") as f:
        lib_hash = f.read().strip()
    res = {"lib_sha256": lib_hash, "bytes": {}, "detail": {},
           "how": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none, last of 3 "
                  "launches of the kernel in `bench.py --workload W --steps 1 --warmup 3` (ncu flushes caches "
                  "before each replayed launch: cold L2)"}
    for spec in sys.argv[1:]:
        w, k = spec.split(":")
        d = capture(w, k)
        res["bytes"][w] = d["bytes"]
        res["detail"][w] = dict(d, kernel=k)
        print(w, d)
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    with open(OUT, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
