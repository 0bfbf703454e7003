#define HXF_P 12
#include "op_inst.cuh"
