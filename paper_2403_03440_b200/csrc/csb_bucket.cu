// csflow-b200: one species bucket of every templated kernel.  build.py
// compiles this file once per bucket with -DCSB_BUCKET=<b>.
#ifndef CSB_BUCKET
#define CSB_BUCKET 6
#endif
#include "csb_rhs.cuh"
#include "csb_implicit.cuh"
#include "csb_sweep.cuh"
#include "csb_update.cuh"
#include "csb_wave.cuh"
