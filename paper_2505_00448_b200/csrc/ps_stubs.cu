// Temporary stubs for kernel families not yet implemented.
#include "ps_internal.cuh"
