// K3 with an 8.8 fixed-point guide (the warped image of the interpolating warp,
// NEXT row f2, reading 21): the same kernel template as
// aggregate_slide.cu instantiated with G16 = true (range factor on the MUFU pipe
// instead of the uint8 difference table), compiled as its own object so the two
// instantiation sets build in parallel.
#define RSR_SLIDE_G16 1
#include "aggregate_slide.cu"
