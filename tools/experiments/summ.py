"""One line per bench JSON file: us/call, roofline fraction, e2e us/call, clocks."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        e = d.get("e2e") or {}
        print(f"{f:40s} {d['us_per_call']:9.2f} us  frac {d['roofline']['frac']:.3f}  e2e {e.get('us_per_call', 0):8.2f} us"
              f"  {d['clocks'].get('sm_mhz')} MHz {d['clocks'].get('reasons')}")
    except Exception as ex:  # noqa: BLE001
        print(f"{f:40s} -- {ex}")
