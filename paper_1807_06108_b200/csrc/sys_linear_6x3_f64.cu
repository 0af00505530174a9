// Engine instantiation: the generic linear plugin f(x) = A x, G constant, B = H = G
// (systems.cuh Linear) with the diagonal quadratic cost, n=6, m=3, double.
#include "engine.cuh"

namespace jm {
EngineBase* make_linear_6x3_f64() { return new Engine<Linear<6, 3>, CostDiagQuadratic, double>(); }
}  // namespace jm
