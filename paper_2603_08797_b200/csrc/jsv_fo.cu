// jsv_fo.cu -- translation unit of the fan-out (star) solver (jsv_fanout.cuh).
#include <cub/block/block_scan.cuh>
#include "jsv_s2common.cuh"
#include "jsv_fanout.cuh"
