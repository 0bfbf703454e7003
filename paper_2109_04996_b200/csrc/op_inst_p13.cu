#define HXF_P 13
#include "op_inst.cuh"
