// Engine instantiation: the generic linear plugin f(x) = A x, G constant, B = H = G
// (systems.cuh Linear) with the diagonal quadratic cost, n=4, m=2, float.
#include "engine.cuh"

namespace jm {
EngineBase* make_linear_4x2_f32() { return new Engine<Linear<4, 2>, CostDiagQuadratic, float>(); }
}  // namespace jm
