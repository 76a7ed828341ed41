#!/bin/bash
# phase stamps of the fused kernel on small layouts, for each probe build given in LIBS
mkdir -p gpurun_out
for lib in ${LIBS:-probe}; do
export CDSGD_LIB=$PWD/paper_2106_10796_b200/libcdsgd_b200_$lib.so
for L in resnet20; do
timeout 300 python scripts/small_probe.py --layout $L --periods 10 --probe --tag ${lib}_$L 2>&1 | tail -1
done
done | tee gpurun_out/${TAG}_probe.jsonl > /dev/null
python - <<PY
import json
for l in open("gpurun_out/${TAG}_probe.jsonl"):
    if not l.startswith("{"): print(l); continue
    d=json.loads(l); p=d['probe']; print(d['tag'], {k:round(v,2) for k,v in d['us_per_step'].items()}, 'span',p['span_ns'], 'start',p['start_ns'],'end',p['end_ns'])
    print('   ', {k[:-4]: v['p50'] for k,v in p.items() if k.endswith('_cyc')})
PY
