# ncu --set full (with source) of the fused points kernel on the bench workload; source page CSV
SEL=${1:-"3, .int.4, .int.5"}
TAG=${2:-m5}
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:score_topk_kernel<.int.$SEL, .int.1>" -s 2 -c 1 -o gpurun_out/pts_full_$TAG \
  python bench.py --steps 2 --warmup 1 --no-baseline > gpurun_out/ncu_pts.log 2>&1; echo ncu=$?
ncu -i gpurun_out/pts_full_$TAG.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/pts_src_$TAG.csv 2>/dev/null; echo src=$?
