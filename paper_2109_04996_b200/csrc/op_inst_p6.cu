#define HXF_P 6
#include "op_inst.cuh"
