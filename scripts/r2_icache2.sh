export CDSGD_LIB=$PWD/paper_2106_10796_b200/libcdsgd_b200_probe.so
for k in 4 100000; do timeout 300 python scripts/small_probe.py --k $k --period 4 --periods 10 --probe --tag k$k | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['probe']; print(d['tag'], d['us_per_step'], {k[:-4]: v['p50'] for k,v in p.items() if k.endswith('_cyc')})"; done
