cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_fo.json 2> gpurun_out/bench_fo.err; echo "rc=$?"
VINF_NO_FUSE_O=1 timeout 900 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_nofo.json 2> gpurun_out/bench_nofo.err; echo "rc=$?"
python - <<'P'
import json
for f in ("gpurun_out/bench_fo.json", "gpurun_out/bench_nofo.json"):
    d = json.load(open(f))
    print(f, round(d["value"]), round(d["ms_per_step"]*1000,1), "e2e", round(d["e2e"]["value"]), "f32", round(d["f32_mode"]["value"]), round(d["f32_mode"]["ms_per_step"]*1000,1), "vc2", round(d["vc2_stack_2300"]["value"]), [round(l["ms"],2) for l in d["vc2_stack_2300"]["levels"]], d["clocks"])
P
