// Instantiation unit: batched scans of 4 queries (ssb_batch_kern.cuh).
#include "ssb_batch_kern.cuh"

template void laq::scan::launch_batch_q<4>(laq_ctx*, const laq::scan::BatchScan&, int, int, int, size_t, int);
