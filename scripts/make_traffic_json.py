"""profiles/traffic_<workload>.json from an ncu `--metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv` capture of one step
(bench.py reads it for the roofline's measured-traffic field)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import traffic

csv_path, workload, raw_name = sys.argv[1], sys.argv[2], sys.argv[3]
step = {"config2": "python scripts/ncu_c2_step.py (one config-2 step, 1024 bit-strings, graph replay)",
        "config4": "python scripts/ncu_c4_path.py config4 (one config-4 path, the bench step)",
        "config5": "python scripts/ncu_c4_path.py config5 (one config-5 path)"}.get(workload, workload)
out = {"source": "ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                 f"dram__bytes_write.sum --clock-control none --csv {step}; summarised by "
                 f"scripts/make_traffic_json.py; raw csv profiles/{raw_name}",
       "workload": workload, "kernels": json.loads(traffic(csv_path))}
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
with open(os.path.join(root, "profiles", f"traffic_{workload}.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out["kernels"], indent=1)[:2000])
