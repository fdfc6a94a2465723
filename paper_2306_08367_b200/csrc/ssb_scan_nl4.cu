// K4 scan kernels for queries joining 4 dimension(s).
#include "ssb_scan_inst.cuh"

LAQ_SCAN_INSTANTIATE(4)
