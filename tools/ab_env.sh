# A/B of a library environment switch through bench.py (short runs, no e2e / cpu baseline):
#   bash tools/ab_env.sh VAR v1 v2 ...   -> gpurun_out/ab.txt (two interleaved reps per value)
mkdir -p gpurun_out
var=$1; shift
for rep in 1 2; do for v in "$@"; do
  env "$var=$v" timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 \
    > "gpurun_out/ab_${v}_$rep.json" 2> "gpurun_out/ab_${v}_$rep.err"
  python - "$var" "$v" "gpurun_out/ab_${v}_$rep.json" >> gpurun_out/ab.txt 2>&1 <<'PY' || tail -3 "gpurun_out/ab_${v}_$rep.err" >> gpurun_out/ab.txt
import json, sys
d = json.load(open(sys.argv[3]))
r = d["roofline"]
print(f"{sys.argv[1]}={sys.argv[2]} {d['value']:.1f} tok/s frac {r['frac']:.4f} "
      f"{r['avg_launch_ms'] * 1e3:.2f} us/launch {d['clocks']['sm_mhz']} MHz")
PY
done; done
cat gpurun_out/ab.txt
