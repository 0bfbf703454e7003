#define HXF_P 14
#include "op_inst.cuh"
