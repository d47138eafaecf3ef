// Throughput instantiation of the cluster bond kernel (k_cluster_impl.cuh):
// 256 threads, two CTAs per SM -- batches of global-slice clusters.  Two
// instances share each SM and hide each other's barrier and memory stalls;
// the per-row state lives in global memory so two carves fit, leaving the
// rest of the unified L1 to the row passes (measured +4% options/s on cfg4
// against one 512-thread CTA per SM, profiles/r01/ab_cta_shape.log).
#define CK_NS ck_tp
#ifndef TP_THREADS
#define TP_THREADS 256
#endif
#ifndef TP_QX_ROWS
#define TP_QX_ROWS 16
#endif
#define CLUSTER_THREADS TP_THREADS
#define CLUSTER_MIN_BLOCKS 2
#define QX_ROWS_DEF TP_QX_ROWS
#include "k_cluster_impl.cuh"
