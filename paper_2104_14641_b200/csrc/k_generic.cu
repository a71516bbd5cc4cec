// Kernel instantiations of one scoring path (compiled as its own translation
// unit so the paths build in parallel); see dev.cuh for the kernels.
#include "dev.cuh"

// MODE 0: generic per-candidate folds; the 4 x 4 layout here, the wide layout in k_generic_wide.cu
ScoreFn k_score_fn_generic_wide(int src);
TopkFn k_topk_fn_generic_wide(int src);
EsGenFn k_es_gen_fn_generic_wide();
ScoreFn k_score_fn_generic(const DTask& T, int src) {
  if (T.layout_rm == 4) return src ? score_kernel<4, 4, 0, 1> : score_kernel<4, 4, 0, 0>;
  return k_score_fn_generic_wide(src);
}
TopkFn k_topk_fn_generic(const DTask& T, int src) {
  if (T.layout_rm == 4) return src ? score_topk_kernel<4, 4, 0, 1> : score_topk_kernel<4, 4, 0, 0>;
  return k_topk_fn_generic_wide(src);
}
EsGenFn k_es_gen_fn_generic(const DTask& T) {
  return T.layout_rm == 4 ? es_gen_kernel<4, 4, 0> : k_es_gen_fn_generic_wide();
}
