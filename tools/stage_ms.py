import json, sys
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
tag = sys.argv[1] if len(sys.argv) > 1 else ""
print(tag, d["ms_per_step"], {k: v["ms"] for k, v in d["stages"].items()})
