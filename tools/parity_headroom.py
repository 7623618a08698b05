"""Summarise a GPU parity log (tests run with VI_PARITY_LOG=<file>) into the headroom table of
profiles/r02_parity_headroom.md: per test (and per attention-kernel check) the worst stage over
all steps, its rel_err, the bar, their ratio, and the distance to the bf16-storage emulation.

    python tools/parity_headroom.py gpurun_out/final/parity_log.jsonl profiles/r02_parity_headroom.md
"""
import json
import sys

HEADER = """# GPU parity headroom (round 2, one B200, `tools/gpu_final.sh main` with VI_PARITY_LOG)

Worst stage of every test over all its steps: rel_err (reading Q18) against the fp64 oracle, the
bar it is held to, their ratio, and (logit-sensitive variants) the GPU's distance to the bf16-storage
emulation (logged, not asserted).  Bars: 2e-2 (bf16) / 1e-4 (fp32) at the paper's N(0, 0.02)
weights; 2e-2 + E for the sensitive / sharp variants, E = emulation vs oracle (GPU-free);
`[attention kernel]` = the attention output against fp64 attention of the GPU's own Q/K/V.

| test | worst stage | rel_err | bar | ratio | vs emulation |
|---|---|---|---|---|---|
"""


def main(src, dst):
    worst = {}
    for line in open(src):
        d = json.loads(line)
        name = d["test"].split("::")[-1]
        if d.get("worst_stage") == "o_kernel":
            name += " [attention kernel]"
        if name not in worst or d["ratio"] > worst[name]["ratio"]:
            worst[name] = d
    rows = []
    for name in sorted(worst):
        d = worst[name]
        emu = d.get("vs_emulation")      # {"stage": worst stage, "err": its distance}
        emu_s = f"{emu['err']:.4f} ({emu['stage']})" if isinstance(emu, dict) and "err" in emu else "-"
        rows.append(f"| {name} | {d['worst_stage']} | {d['err']:.4f} | {d['bar']:.4f} | {d['ratio']:.2f} | {emu_s} |")
    mx = max(worst.values(), key=lambda d: d["ratio"])
    with open(dst, "w") as f:
        f.write(HEADER + "\n".join(rows) + "\n")
        f.write(f"\n{len(worst)} checks; largest ratio {mx['ratio']:.2f} ({mx['test'].split('::')[-1]}, "
                f"{mx['worst_stage']}).\n")
    print(f"{len(worst)} checks -> {dst}; max ratio {mx['ratio']:.2f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
