#define HXF_P 11
#include "op_inst.cuh"
