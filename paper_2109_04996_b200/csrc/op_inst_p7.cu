#define HXF_P 7
#include "op_inst.cuh"
