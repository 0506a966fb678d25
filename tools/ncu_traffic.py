"""Per-launch DRAM traffic of the decode-step kernels from one `ncu --set full` capture.

    python tools/ncu_traffic.py profiles/r01/ncu_kernels.csv > profiles/r01/ncu_traffic.json

Input: `ncu -i prof.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,...`
(profiles/gpu_round.sh captures the report).  Output: {stage: {"kernel", "traffic_bytes",
"duration_us"}} keyed by the bench.py stage names, so bench.py can put the measured
dram__bytes_read.sum + dram__bytes_write.sum of the dominant kernel into roofline.traffic.
"""

import csv
import json
import sys

STAGES = {"front_half_kernel": "mac_match_scan", "front_bf16_d128_kernel": "mac_match_scan",
          "verify_kernel": "mac_match_verify", "amend_mma_kernel": "mac_amend", "amend_tma_kernel": "mac_amend",
          "dense_kernel": "mac_match_verify", "complete_bf16_kernel": "mac_complete"}
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    ix = {k: hdr.index(k) for k in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                    "gpu__time_duration.sum")}
    acc = {}
    for r in rows[2:]:
        name = r[ix["Kernel Name"]]
        stage = next((s for k, s in STAGES.items() if k in name), None)
        if stage is None:
            continue
        b = sum(float(r[ix[m]].replace(",", "")) * UNIT[units[ix[m]]]
                for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        us = float(r[ix["gpu__time_duration.sum"]].replace(",", ""))
        acc.setdefault(stage, []).append((name, b, us))
    out = {s: {"kernel": v[0][0], "traffic_bytes": sum(x[1] for x in v) / len(v),
               "duration_us": sum(x[2] for x in v) / len(v), "launches": len(v)} for s, v in acc.items()}
    out["_source"] = f"ncu --set full --clock-control none capture ({path}); dram__bytes_read.sum + dram__bytes_write.sum per launch"
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1])
