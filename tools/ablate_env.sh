#!/usr/bin/env bash
# Each library ablation switch against the default, one bench run each (c2-inner, 1 GPU).
# Usage: bash tools/ablate_env.sh > profiles/r1_ablation.jsonl
set -u
run() {
  local tag="$1"; shift
  local out
  out=$(env "$@" timeout -s KILL 120 python bench.py --no-cpu-baseline 2>/dev/null | tail -1)
  python - "$tag" "$out" <<'PY'
import json, sys
tag, line = sys.argv[1], sys.argv[2]
try:
    d = json.loads(line)
    print(json.dumps({"switch": tag, "ms_per_step": round(d["ms_per_step"], 4), "samples_per_s": round(d["value"]),
                      "e2e_samples_per_s": round(d["e2e"]["value"]),
                      "kernels_ms": {k: round(v["ms_per_launch"], 4) for k, v in d["kernels"].items()},
                      "sections_ms": {k: round(v["ms"], 4) for k, v in d["sections"].items()}}))
except Exception as e:
    print(json.dumps({"switch": tag, "error": str(e)[:200]}))
PY
}
run default X=1
run LONGER_HEAD_ROWS=0 LONGER_HEAD_ROWS=0
run LONGER_INNER_NG=1 LONGER_INNER_NG=1
run LONGER_GEMM_STAGE=0 LONGER_GEMM_STAGE=0
run LONGER_SPLIT_ITEMS=296 LONGER_SPLIT_ITEMS=296
run LONGER_ATTN_TMA=0 LONGER_ATTN_TMA=0
run LONGER_ATTN_PACK=0 LONGER_ATTN_PACK=0
run LONGER_ITEM_SMEM=0 LONGER_ITEM_SMEM=0
run LONGER_PRIO=0 LONGER_PRIO=0
run LONGER_PDL=0 LONGER_PDL=0
run LONGER_SIDE=0 LONGER_SIDE=0
run LONGER_LN_LEAN=0 LONGER_LN_LEAN=0
run LONGER_LN_ASYNC=0 LONGER_LN_ASYNC=0
run LONGER_LN_ASYNC=1 LONGER_LN_ASYNC=1
run LONGER_LN_RPB=16 LONGER_LN_RPB=16
run LONGER_ATTN_TC=0 LONGER_ATTN_TC=0
run LONGER_FUSED=0 LONGER_FUSED=0
run default_again X=1
