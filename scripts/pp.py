import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(sys.argv[1], round(d["ms_per_step"],2), [p["ms"] for p in d["roofline"]["per_pass"]])
