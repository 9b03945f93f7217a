// Explicit instantiation unit: dtype float, 2-D grids (all features, parametrisations, KP).
#include "launch.cuh"
namespace sr {
SR_DEFINE_INST(f32, float, 2)
}  // namespace sr
