// placeholder: tcgen05 GEMM lands here
#include "sf_internal.h"
