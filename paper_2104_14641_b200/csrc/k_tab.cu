// Kernel instantiations of one scoring path (compiled as its own translation
// unit so the paths build in parallel); see dev.cuh for the kernels.
#include "dev.cuh"

// MODE 1 / 2: tabulated dimension counts (table in global / shared memory); MODE 3: tensor
// tables (points) -- DESIGN.md §3.5.  MODE 2 (the common one) lives in k_tab2.cu.
ScoreFn k_score_fn_tab2(int src);
TopkFn k_topk_fn_tab2(int src);
EsGenFn k_es_gen_fn_tab2();
ScoreFn k_score_fn_tab(const DTask& T, int mode, int src) {
  if (src && mode == 3) return score_kernel<4, 4, 3, 1>;
  if (mode == 1) return src ? score_kernel<4, 4, 1, 1> : score_kernel<4, 4, 1, 0>;
  return k_score_fn_tab2(src);
}
TopkFn k_topk_fn_tab(const DTask& T, int mode, int src) {
  if (src && mode == 3) return score_topk_kernel<4, 4, 3, 1>;
  if (mode == 1) return src ? score_topk_kernel<4, 4, 1, 1> : score_topk_kernel<4, 4, 1, 0>;
  return k_topk_fn_tab2(src);
}
EsGenFn k_es_gen_fn_tab(const DTask& T, int mode) {
  if (mode == 3) return es_gen_kernel<4, 4, 3>;
  if (mode == 2) return k_es_gen_fn_tab2();
  return es_gen_kernel<4, 4, 1>;
}
