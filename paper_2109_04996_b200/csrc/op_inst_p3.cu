#define HXF_P 3
#include "op_inst.cuh"
