// Engine instantiation: the generic linear plugin f(x) = A x, G constant, B = H = G
// (systems.cuh Linear) with the diagonal quadratic cost, n=2, m=1, double.
#include "engine.cuh"

namespace jm {
EngineBase* make_linear_2x1_f64() { return new Engine<Linear<2, 1>, CostDiagQuadratic, double>(); }
}  // namespace jm
