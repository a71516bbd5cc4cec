// Kernel instantiations of one scoring path (compiled as its own translation
// unit so the paths build in parallel); see dev.cuh for the kernels.
#include "dev.cuh"

// MODE 0, wide layout (up to MAXT tensors x MAXRANK dimensions)
ScoreFn k_score_fn_generic_wide(int src) {
  return src ? score_kernel<MAXT, MAXRANK, 0, 1> : score_kernel<MAXT, MAXRANK, 0, 0>;
}
TopkFn k_topk_fn_generic_wide(int src) {
  return src ? score_topk_kernel<MAXT, MAXRANK, 0, 1> : score_topk_kernel<MAXT, MAXRANK, 0, 0>;
}
EsGenFn k_es_gen_fn_generic_wide() { return es_gen_kernel<MAXT, MAXRANK, 0>; }
