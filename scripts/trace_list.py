"""Print the kernel/memcpy list of a Chrome trace written by scripts/timeline.py (stream, start, duration)."""
import json
import sys

ev = json.load(open(sys.argv[1]))["traceEvents"]
ks = sorted((e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")),
            key=lambda e: e["ts"])
t0 = ks[0]["ts"]
for e in ks[int(sys.argv[2]) if len(sys.argv) > 2 else 0:]:
    print(f"{e['ts'] - t0:9.1f} {e['dur']:8.1f} s{e['args'].get('stream'):<4} {e['name'][:70]}")
