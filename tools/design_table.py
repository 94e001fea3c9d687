"""Markdown rows of DESIGN.md §7's round table from profiles/<round>/bench_*.json
(after tools/refresh_profiles.py).   python tools/design_table.py [round2]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1] if len(sys.argv) > 1 else "round2"
NAMES = {
    "cfg2": "cfg2 multipeak8 d=8, 1e8/it (headline)",
    "cfg1": "cfg1 gaussian d=4, 1e6/it, ng=1000",
    "cfg3": "cfg3 ridge d=4, 1e8/it",
    "cfg4a": "cfg4a genz oscillatory d=6, 1e9/it",
    "cfg4b": "cfg4b genz product-peak d=6, 1e9/it",
    "cfg5": "cfg5 gaussian20 d=20, 4e9/it (split fill)",
    "ra10": "ra10 Roos & Arnold d=10, 5e8/it (the paper's workload)",
}
ROUND1 = {"cfg2": "2.99e10", "cfg1": "9.39e9", "cfg3": "5.98e9", "cfg4a": "4.14e10",
          "cfg4b": "4.34e10", "cfg5": "1.14e10", "ra10": "2.47e10"}


def g(x):
    return f"{x:.3g}".replace("e+0", "e").replace("e+", "e")


for c, name in NAMES.items():
    d = json.load(open(os.path.join(ROOT, "profiles", rnd, f"bench_{c}.json")))
    r = d["roofline"]
    fr = f"{r['frac']:.3f}"
    sv = r.get("frac_survey_figure")
    if sv and abs(sv - r["frac"]) > 0.002:
        fr += f" [{sv:.3f}]" if sv < 2 else f" [{sv:.1f}]"
    print(f"| {name} | {g(d['value'])} | {fr} | {r['issue']['frac']:.2f} | "
          f"{d['ms_per_step']:.3g} | {g(d['cpu_baseline']['value'])} | {g(d['e2e']['value'])} | "
          f"{ROUND1[c]} |")
