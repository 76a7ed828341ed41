#!/bin/bash
# same-kernel sequences (no correction rounds: k large) vs the k=4 mix
for k in 4 100000; do timeout 300 python scripts/small_probe.py --k $k --period 4 --periods 10 --tag k$k | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['tag'], d['us_per_step'])"; done
