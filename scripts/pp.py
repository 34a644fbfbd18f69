"""Prints ms/step and the per-pass times of a bench.py JSON line read from stdin.
usage: python bench.py ... | python scripts/pp.py <label>"""
import json, sys

d = json.loads(sys.stdin.read().strip().splitlines()[-1])
print(sys.argv[1] if len(sys.argv) > 1 else "-", round(d["ms_per_step"], 2), [p["ms"] for p in d["roofline"]["per_pass"]])
