"""Predicted maximum trainable context per SP size (planner.py) next to the measured
single-GPU frontier.  Prints one JSON document (profiles/max_context_model_r02.json)."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2604_27089_b200.planner import predict_max_context, step_memory  # noqa: E402
from paper_2604_27089_b200.workloads import CONFIGS  # noqa: E402

DEVICE = 178.35 * 2 ** 30  # B200 capacity as reported by the driver (torch total_memory)
measured = {}
try:
    m = json.loads((ROOT / "profiles" / "max_context_r01_llama3-8b_n1.json").read_text())
    measured[("llama3-8b", 1)] = m["max_trainable_seq"]
except Exception:
    pass
out = {"device_bytes": DEVICE, "model": "paper_2604_27089_b200/planner.py (auto_sp + sp_ac "
       "seq-aware + ZeRO-1 for P > 1)", "rows": []}
for name in ("llama3-8b", "llama3.2-1b"):
    cfg = CONFIGS[name]
    for P in (1, 2, 4, 8):
        s = predict_max_context(cfg, P, DEVICE)
        est = step_memory(cfg, s, P)
        out["rows"].append({"model": name, "sp": P, "predicted_max_seq": s,
                            "measured_max_seq": measured.get((name, P)),
                            "at_prediction_gb": {"static": round(est.static / 1e9, 1),
                                                 "saved": round(est.saved / 1e9, 1),
                                                 "symmetric_heap": round(est.pool / 1e9, 1),
                                                 "transient": round(est.transient / 1e9, 1)}})
print(json.dumps(out, indent=1))
