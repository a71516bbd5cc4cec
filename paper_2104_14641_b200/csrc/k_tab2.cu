// Kernel instantiations of one scoring path (compiled as its own translation
// unit so the paths build in parallel); see dev.cuh for the kernels.
#include "dev.cuh"

// MODE 2: tabulated dimension counts, table in shared memory -- the records path
ScoreFn k_score_fn_tab2(int src) { return src ? score_kernel<4, 4, 2, 1> : score_kernel<4, 4, 2, 0>; }
TopkFn k_topk_fn_tab2(int src) { return src ? score_topk_kernel<4, 4, 2, 1> : score_topk_kernel<4, 4, 2, 0>; }
EsGenFn k_es_gen_fn_tab2() { return es_gen_kernel<4, 4, 2>; }
