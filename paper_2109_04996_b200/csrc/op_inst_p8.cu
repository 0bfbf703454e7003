#define HXF_P 8
#include "op_inst.cuh"
