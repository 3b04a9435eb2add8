"""DESIGN.md section 9 table from the clocked bench lines of one evidence tag (profiles/<tag>_bench_*.json)."""
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r02g"
order = ["tiny", "small", "medium_h64", "medium_h32", "medium_h16", "medium_h8", "large", "large_per_pair",
         "large_ctf4", "large_fast", "translations", "translations_landscape"]
label = {"tiny": "Tiny", "small": "Small", "large": "Large", "large_per_pair": "Large", "large_ctf4": "Large, 4 CTF groups",
         "large_fast": "Large, fast (2e-3)", "translations": "Translations", "translations_landscape": "Translations"}
print("| Config | H | mode | step ms | align ms | contraction ms | transform ms | compress ms | partials ms | pairs/s | step / align roofline frac | clocks |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|")
for name in order:
    f = os.path.join(ROOT, "profiles", f"{tag}_bench_{name}.json")
    if not os.path.exists(f):
        continue
    d = json.loads(open(f).read())
    c, ph, sr, ck = d["config"], d["phases_ms_last_step"], d["step_roofline"], d.get("clocks", {})
    k = sr.get("kernel_ms_per_step", {})
    mode = {"per_pair": "per pair", "per_image": "per image", "landscape": "landscape"}[c["mode"]]
    if name == "translations_landscape":
        mode += " (77.3 GB streamed)"
    lab = label.get(name, "Medium")
    mhz = ck.get("sm_mhz")
    clk = "too short to sample" if mhz is None else f"{mhz:.0f} MHz" + (", " + ", ".join(ck.get("reasons", [])) if ck.get("reasons") else "")
    print(f"| {lab} | {c['H']} | {mode} | {d['ms_per_step']:.2f} | {ph.get('align', 0):.2f} | {k.get('contract', 0):.2f} | "
          f"{k.get('fft_reduce', 0):.2f} | {k.get('compress', 0):.2f} | {k.get('kernel_partials', 0):.2f} | {d['value']:.3g} | "
          f"{sr['frac']:.2f} / {sr['frac_align_only']:.2f} | {clk} |")
