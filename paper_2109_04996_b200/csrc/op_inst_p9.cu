#define HXF_P 9
#include "op_inst.cuh"
