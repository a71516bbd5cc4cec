// Kernel instantiations of one scoring path (compiled as its own translation
// unit so the paths build in parallel); see dev.cuh for the kernels.
#include "dev.cuh"

// MODE 6: general trees
ScoreFn k_score_fn_tree(int src) { return src ? score_kernel<4, 4, 6, 1> : score_kernel<4, 4, 6, 0>; }
TopkFn k_topk_fn_tree(int src) { return src ? score_topk_kernel<4, 4, 6, 1> : score_topk_kernel<4, 4, 6, 0>; }
EsGenFn k_es_gen_fn_tree() { return es_gen_kernel<4, 4, 6>; }
