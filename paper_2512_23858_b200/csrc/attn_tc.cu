// tcgen05 tree attention (bf16) — placeholder until written
#include "common.cuh"
#include "host_util.h"
extern "C" int ygg_prepare_attn_tc(void) { return YGG_OK; }
