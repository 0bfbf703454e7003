#define HXF_P 5
#include "op_inst.cuh"
