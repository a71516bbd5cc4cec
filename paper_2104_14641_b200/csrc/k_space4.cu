// Kernel instantiations of one scoring path (compiled as its own translation
// unit so the paths build in parallel); see dev.cuh for the kernels.
#include "dev.cuh"

// MODE 4: space-specialised points path, 64-bit walk
ScoreFn k_score_fn_space4(const DTask& T) {
  switch (T.n_tensors) {
    case 1: return score_kernel<1, 4, 4, 1>;
    case 2: return score_kernel<2, 4, 4, 1>;
    case 3: return score_kernel<3, 4, 4, 1>;
    default: return score_kernel<4, 4, 4, 1>;
  }
}
TopkFn k_topk_fn_space4(const DTask& T, int src) {  // src 2: points in mapped pinned host memory
  switch (T.n_tensors) {
    case 1: return src == 2 ? score_topk_kernel<1, 4, 4, 2> : score_topk_kernel<1, 4, 4, 1>;
    case 2: return src == 2 ? score_topk_kernel<2, 4, 4, 2> : score_topk_kernel<2, 4, 4, 1>;
    case 3: return src == 2 ? score_topk_kernel<3, 4, 4, 2> : score_topk_kernel<3, 4, 4, 1>;
    default: return src == 2 ? score_topk_kernel<4, 4, 4, 2> : score_topk_kernel<4, 4, 4, 1>;
  }
}
EsGenFn k_es_gen_fn_space4(const DTask& T) {
  switch (T.n_tensors) {
    case 1: return es_gen_kernel<1, 4, 4>;
    case 2: return es_gen_kernel<2, 4, 4>;
    case 3: return es_gen_kernel<3, 4, 4>;
    default: return es_gen_kernel<4, 4, 4>;
  }
}
