"""profiles/traffic.json from ncu --set full captures: DRAM bytes (read +
write) per cell of each sweep, keyed like bench.py looks them up
(<workload>_<flux>_<math>_sweep_<x|y|xy>_dram_bytes_per_cell; xy = the fused step).
    python tools/traffic_json.py cfg3_hllc_tolerance=rep1 cfg3_hllc_bitwise=rep2 ..."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import kernel_metrics  # noqa: E402

CELLS = {"cfg0": 256 ** 2, "cfg1": 2048 ** 2, "cfg2": 8192 ** 2, "cfg3": 16384 ** 2, "cfg4": 16384 ** 2}
out = {"source": "ncu --set full --clock-control none (tools/r2k_final.sh captures: the fused step on config 3, "
                 "one column and one row sweep on config 2): (dram__bytes_read.sum + dram__bytes_write.sum) / cells",
       "alg_bytes_per_cell": 64}
for arg in sys.argv[1:]:
    key, rep = arg.split("=", 1)
    cells = CELLS[key.split("_")[0]]
    for k in kernel_metrics(rep, cells):
        if "sweep" not in k["kernel"] or "dram_bytes" not in k:
            continue
        which = "xy" if "sweep_xy" in k["kernel"] else ("x" if "sweep_x" in k["kernel"] else "y")
        out[f"{key}_sweep_{which}_dram_bytes_per_cell"] = round(k["dram_bytes"] / cells, 3)
json.dump(out, open("profiles/traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
