python tools/trace_topk.py 2>&1 | grep LS_TRACE | tail -8
