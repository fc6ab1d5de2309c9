# A/B/... the step time: alternate env settings within one box session (clocks drift between
# boxes).  usage: R=2 ARGS="--layers 16" bash tools/ab.sh "ENV_A" "ENV_B" ...
R="${R:-2}"
mkdir -p gpurun_out
for i in $(seq 1 $R); do
  for cfg in "$@"; do
    out=$(env $cfg python bench.py --no-cpu-baseline --no-e2e $ARGS 2>/dev/null | tail -1)
    python - "$cfg" "$out" <<'PY'
import json, sys
cfg, line = sys.argv[1], sys.argv[2]
try:
    d = json.loads(line)
except Exception:
    print(cfg, "FAILED", line[:200]); sys.exit()
L = d["config"]["layers"]
sh = {k[:-5] if k.endswith("_gemm") else k: v for k, v in d["kernel_us_per_layer"].items()}
sh["rest"] = round(d["ms_per_step"] * 1000 / L - sum(sh.values()), 1)
print(f"{cfg:44s} {d['ms_per_step']:.3f} ms sm {d['clocks']['sm_mhz']} {d['clocks']['reasons']} {sh}")
PY
  done
done
