#define HXF_P 16
#include "op_inst.cuh"
