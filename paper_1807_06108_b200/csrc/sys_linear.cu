// Engine instantiations for the generic linear plugin f(x) = A x, G constant,
// B = H = G (systems.cuh Linear), with the diagonal quadratic cost.
#include "engine.cuh"

namespace jm {
template <int N, int M>
EngineBase* make_linear(int precision) {
  if (precision == JM_F64) return new Engine<Linear<N, M>, CostDiagQuadratic, double>();
  return new Engine<Linear<N, M>, CostDiagQuadratic, float>();
}

EngineBase* make_engine_linear(int cost_kind, int precision, int n, int m) {
  if (cost_kind != JM_COST_DIAG_QUADRATIC) return nullptr;
  if (n == 2 && m == 1) return make_linear<2, 1>(precision);
  if (n == 4 && m == 1) return make_linear<4, 1>(precision);
  if (n == 4 && m == 2) return make_linear<4, 2>(precision);
  if (n == 6 && m == 3) return make_linear<6, 3>(precision);
  return nullptr;
}
}  // namespace jm
