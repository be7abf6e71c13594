// paces_b200.cu -- unity translation unit of libpaces_b200.so (kernels are defined once, in headers).
#include "engine.cu"
#include "incremental.cu"
#include "sharded.cu"
#include "capi.cu"
