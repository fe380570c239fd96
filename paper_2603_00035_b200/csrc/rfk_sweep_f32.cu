// rfk_sweep_f32.cu — the fp32 mode of the sweep: the same
// wavefront kernel as rfk_sweep.cu, instantiated with fp32 storage and
// arithmetic.  Records are hoisted in fp64 (rfk_sweep.cu's hoist_kernel) and
// rounded; parity target: 1e-4 relative to the fp64 oracle.
#define RFK_SWEEP_F32 1
#include "rfk_sweep.cu"
