"""Convert tools/pipe_bench output (warp-instr/cycle/SM per instruction mix)
into the ACS roofline denominators recorded in profiles/acs_peak.json."""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.startswith("{") and "op" in l]
best = {}
for r in rows:
    best[r["op"]] = max(best.get(r["op"], 0.0), r["warp_instr_per_cycle_per_sm"])
s32 = best["ACS2_s32(IMAD+VIADDMNMX)"] / 2 * 32        # 2 instr per state update, 32 lanes
u16 = best["ACS2_u16x2(VIADD16x2+VIADDMNMX)"] / 2 * 2 * 32  # 2 instr per 2 state updates
out = {
    "source": "tools/pipe_bench.cu on one B200 (gpurun), best over 4..32 warps/SM",
    "warp_instr_per_cycle_per_sm": best,
    "state_updates_per_cycle_per_sm": {"s32_imad_viaddmnmx": s32, "u16x2_viadd_viaddmnmx": u16},
    "note": "one radix-2 state update = candidate add (IMAD or VIADD.16x2) + fused add-max (VIADDMNMX); the "
            "u16x2 form updates two states per instruction pair and is the roofline peak used by bench.py",
}
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out["state_updates_per_cycle_per_sm"]))
