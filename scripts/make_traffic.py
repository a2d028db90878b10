"""profiles/roofline_traffic.json from committed-capture reports: per-launch
DRAM bytes, L2 bytes (lts__t_sectors x 32) and shared-memory wavefronts of the
dominant kernel of each bench config, read by bench.py (measured_traffic).

usage: python scripts/make_traffic.py "KEY|REPORT|UPDATES|LAUNCHES_PER_STEP|SOURCE_TXT" ...
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import values  # noqa: E402

out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                        "roofline_traffic.json")
doc = json.load(open(out_path)) if os.path.exists(out_path) else {}
for arg in sys.argv[1:]:
    key, rep, upl, lps, src = arg.split("|", 4)
    h, u, v, d = values(rep)
    doc[key] = {
        "dram_bytes_per_launch": d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0),
        "lts_bytes_per_launch": 32 * d.get("lts__t_sectors.sum", 0),
        "smem_wavefronts_per_launch": d.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 0),
        "updates_per_launch": int(float(upl)),
        "launches_per_step": int(lps),
        "ncu_kernel": v[h.index("Kernel Name")],
        "source": src,
    }
json.dump(doc, open(out_path, "w"), indent=1)
print(json.dumps(doc, indent=1)[:400])
