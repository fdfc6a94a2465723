// K4 scan kernels for queries joining 5 dimension(s).
#include "ssb_scan_inst.cuh"

LAQ_SCAN_INSTANTIATE(5)
