# A/B of an environment setting on one box: the default 8B bench (A) against the same with
# "$@" exported (B), alternating three times (the power-capped clock drifts between runs).
#   bash scripts/ab_env.sh CFT_GEMM_GROUP_LONGK=8
run() { timeout 900 env "$@" python bench.py --gpus 1 --steps 20 --warmup 5 --no-sweep --no-cpu-baseline 2>/dev/null | tail -1; }
for i in 1 2 3; do
  A=$(run CFT_AB_TAG=A)
  B=$(run "$@")
  python - "$A" "$B" <<'PY'
import json, sys
for tag, line in zip("AB", sys.argv[1:]):
    d = json.loads(line)
    p = d["phases_ms_per_step"]
    print(tag, round(d["value"]), round(d["ms_per_step"], 2), d["clocks"]["sm_mhz"],
          round(d["value"] / d["clocks"]["sm_mhz"], 2),
          {k: round(v, 2) for k, v in p.items() if k in ("fwd_gemm", "dgrad", "wgrad")})
PY
done
