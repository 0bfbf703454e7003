#define HXF_P 2
#include "op_inst.cuh"
