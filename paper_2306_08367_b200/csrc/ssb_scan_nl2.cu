// K4 scan kernels for queries joining 2 dimension(s).
#include "ssb_scan_inst.cuh"

LAQ_SCAN_INSTANTIATE(2)
