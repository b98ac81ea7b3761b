"""Print value + per-stage (ms, roofline fraction) of bench JSON lines."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["value"], {k: (v["ms"], v.get("frac")) for k, v in d["stages"].items()})
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable:", e)
