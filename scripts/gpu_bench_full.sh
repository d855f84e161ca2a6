cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
python - <<'PY'
import json; d=json.load(open('gpurun_out/bench_full.json'))
print("value", round(d["value"]), "ms/step", round(d["ms_per_step"],4), "e2e", round(d["e2e"]["value"]))
v=d["vc2_stack_2300"]; print("vc2", round(v["value"]), v["ms_per_step"], [round(l["ms"],2) for l in v["levels"]], v["clocks"])
print("f32", round(d["f32_mode"]["value"]))
PY
