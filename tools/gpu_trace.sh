# phase timestamps of the fused kernel at 2^20 / 2^22 (LS_TRACE=1), per-block main-loop ends
LS_TRACE_BLOCKS=1 timeout 300 python tools/trace_topk.py > gpurun_out/trace.log 2>&1; echo trace=$?
