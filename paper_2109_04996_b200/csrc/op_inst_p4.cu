#define HXF_P 4
#include "op_inst.cuh"
