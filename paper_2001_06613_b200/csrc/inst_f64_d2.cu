// Explicit instantiation unit: dtype double, 2-D grids (all features, parametrisations, KP).
#include "launch.cuh"
namespace sr {
SR_DEFINE_INST(f64, double, 2)
}  // namespace sr
