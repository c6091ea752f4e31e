// bsg_internal.h — declarations shared between the CUDA C-ABI (bsg_capi.cu)
// and the host C++ closed-loop driver (bsg_driver.cpp).
#pragma once

#include "../../include/blocksim_b200.h"

#ifdef __cplusplus
/* validate_instance_config (types.cpp:47-61) + the supported integer domain:
 * BSG_OK, BSG_BAD_CONFIG (*field_code = bsg_set_configs' field code) or
 * BSG_BAD_INPUT. Shared by bsg_set_configs and the wire codec. */
bsg_status bsg_check_config(const bsg_instance_cfg& c, int32_t* field_code);
#endif
