// Temporary stubs for kernel families not yet implemented.
#include "ps_internal.cuh"
int ps_rank_mixed_run(int, ps_matrix*, ps_matrix*, int64_t, int64_t, int, double*, double*, double*, cudaStream_t) { return ps_fail(PS_ERR_INVALID, "not implemented"); }
