#define HXF_P 15
#include "op_inst.cuh"
