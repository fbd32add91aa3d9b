"""Render tools/config_table.py JSONL as a markdown table."""
import json
import sys

print("| config | instances | pairs | forward ms (fps) | native ms | SW-B t | SW-B ms | speedup |"
      " SW-B G contrib/s | native % of L2 same-addr RED peak | SW-B % of 9-lane RED peak |"
      " SW-B % HBM |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|")
for line in open(sys.argv[1]):
    d = json.loads(line)
    print(f"| {d['config']} | {d['instances']:,} | {d['pairs']:,} | {d['forward_ms']:.3f} "
          f"({d['forward_fps']:.0f}) | {d['native_ms']:.3f} | {d['sw_b_threshold']} | "
          f"{d['sw_b_ms']:.3f} | {d['speedup']:.2f}x | {d['sw_b_contrib_per_s'] / 1e9:.0f} | "
          f"{100 * d['native_l2_red_frac']:.0f} | {100 * d['sw_b_l2_red_frac']:.0f} | "
          f"{100 * d['sw_b_hbm_frac']:.1f} |")
