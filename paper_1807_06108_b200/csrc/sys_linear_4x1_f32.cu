// Engine instantiation: the generic linear plugin f(x) = A x, G constant, B = H = G
// (systems.cuh Linear) with the diagonal quadratic cost, n=4, m=1, float.
#include "engine.cuh"

namespace jm {
EngineBase* make_linear_4x1_f32() { return new Engine<Linear<4, 1>, CostDiagQuadratic, float>(); }
}  // namespace jm
