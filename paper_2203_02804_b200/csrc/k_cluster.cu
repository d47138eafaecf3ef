// Latency instantiation of the cluster bond kernel (k_cluster_impl.cuh):
// 512 threads, one CTA per SM -- single options and small batches, where one
// instance's critical path is the whole wall time.
#define CK_NS ck_lat
#define CLUSTER_THREADS 512
#define CLUSTER_MIN_BLOCKS 1
#define QX_ROWS_DEF 64
#include "k_cluster_impl.cuh"
