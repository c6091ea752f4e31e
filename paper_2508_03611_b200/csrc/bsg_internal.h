// bsg_internal.h — declarations shared between the CUDA C-ABI (bsg_capi.cu)
// and the host C++ closed-loop driver (bsg_driver.cpp).
#pragma once

#include "../../include/blocksim_b200.h"
