// jsv_exh.cu -- translation unit of the exhaustive Stage-2 sweep (jsv_exhaustive.cuh).
#include "jsv_s2common.cuh"
#include "jsv_exhaustive.cuh"
