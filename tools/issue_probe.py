"""FP64 issue-slot probe (ffcu_fp64_issue_probe): DFMA rate with K integer multiply-adds issued per
eight DFMAs, against the two models -- 16 / (16 + K) (an FP64 warp instruction holds the dispatch
for two cycles, nothing issues in its shadow) and min(1, 16 / (8 + K)) (one issue per cycle,
FP64 pipe busy two cycles per instruction, the others alongside)."""
import json
import sys

sys.path.insert(0, ".")
import paper_2003_12875_b200 as fb  # noqa: E402

base = None
rows = []
for k in (0, 2, 4, 5, 6, 8, 16):
    best = max(fb.fp64_issue_probe(k) for _ in range(3))
    base = base or best
    rows.append({"others_per_8_dfma": k, "dfma_per_s": best, "relative": best / base,
                 "model_shadow_blocked": 16 / (16 + k), "model_dual_issue": min(1.0, 16 / (8 + k))})
print(json.dumps({"nominal_dfma_per_s": 148 * 64 * 1.965e9, "rows": rows}, indent=1))
