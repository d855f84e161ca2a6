"""profiles/ncu_traffic.json from a summarize_ncu.py output (the --set full JSON lines):
per kernel group, dram read + write bytes of one launch (bench.py's roofline `traffic`)."""
import json
import sys

GROUPS = {
    # (bf16 out, residual, statistics, TMA epilogue) flavours of gemm_tc_kernel<BN, ...>
    ", 1, 1, 1, 0>": "conv_gemm",
    "colpart_fold": "gn_stats",
    "group_fold_kernel": "gn_fold",
    "group_apply_bf16_kernel": "gn_apply",
    "<240, 1, 0, 0, 1>": "qkv_gemm",
    "<224, 1, 0, 0, 1>": "wvo_gemm",
    "attention_core_kernel": "attn_core",
    ", 1, 1, 0, 1>": "o_gemm",
    "stub_bf16_kernel": "stub",
}
summary, source = sys.argv[1], sys.argv[2]
out = {}
for line in open(summary):
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    for pat, g in GROUPS.items():
        if pat in d["kernel"] and g not in out:
            out[g] = {"dram_bytes": int(round((d["dram_read_MB"] + d["dram_write_MB"]) * 1e6)),
                      "ncu_time_us": d["time_us"], "source": source}
json.dump(out, open("profiles/ncu_traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
