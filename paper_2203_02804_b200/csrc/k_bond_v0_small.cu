// One-CTA bond kernel, small shape (128 threads, 8 CTAs per SM): blocks of at
// most V0_SMALL_BYTES (k_bond_v0.cu dispatches).
#define V0_NS v0_small
#define V0_THREADS 128
#define V0_MIN_BLOCKS 8
#include "k_bond_v0_impl.cuh"
