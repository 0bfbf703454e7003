#define HXF_P 10
#include "op_inst.cuh"
