# A/B of two builds of the library on one box: the working tree's build (B) against
# ab/libchunkft_b200_base.so (A), each through the default 8B bench (no sweep / CPU leg).
run() { timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --no-sweep --no-cpu-baseline 2>/dev/null | tail -1; }
B=$(run)
cp paper_2605_21177_b200/_native/libchunkft_b200.so /tmp/lib_b.so
cp ab/libchunkft_b200_base.so paper_2605_21177_b200/_native/libchunkft_b200.so
A=$(run)
cp /tmp/lib_b.so paper_2605_21177_b200/_native/libchunkft_b200.so
python - "$A" "$B" <<'PY'
import json, sys
for tag, line in zip("AB", sys.argv[1:]):
    d = json.loads(line)
    p = d["phases_ms_per_step"]
    print(tag, round(d["value"]), round(d["ms_per_step"], 2), d["clocks"]["sm_mhz"],
          {k: round(v, 3) for k, v in p.items() if k in ("fwd_other", "bwd_other", "attn_fwd", "attn_bwd", "loss", "update")})
PY
