# A/B of an environment switch (VAR=a,b): the bench and a trace per value, interleaved
VAR=${VAR:-LS_SD_SINGLE}
for r in 1 2 3; do for v in ${VALS:-0 1}; do
  env $VAR=$v timeout 300 python bench.py --no-baseline 2>/dev/null | tail -1 | python -c "
import sys, json; d = json.loads(sys.stdin.read())
print('$VAR=$v', round(d['value'] / 1e9, 3), round(d['e2e']['value'] / 1e9, 3), round(d['ms_per_step'] * 1e3, 1))"
done; done
for v in ${VALS:-0 1}; do env $VAR=$v LS_TRACE=1 timeout 300 python tools/trace_topk.py 2>&1 | grep LS_TRACE | sed -n '3p;6p' | cut -c1-120; done
