// Engine instantiations for the control-channel integrator dx = u dt + eps sqrt(dt)
// (tests/conftest.py:19-30 scalar_integrator; n = m in {1, 2}).
#include "engine.cuh"

namespace jm {
EngineBase* make_engine_integrator(int cost_kind, int precision, int n) {
  if (cost_kind != JM_COST_DIAG_QUADRATIC) return nullptr;
  const bool f64 = precision == JM_F64;
  if (n == 1) {
    if (f64) return new Engine<Integrator<1>, CostDiagQuadratic, double>();
    return new Engine<Integrator<1>, CostDiagQuadratic, float>();
  }
  if (n == 2) {
    if (f64) return new Engine<Integrator<2>, CostDiagQuadratic, double>();
    return new Engine<Integrator<2>, CostDiagQuadratic, float>();
  }
  return nullptr;
}
}  // namespace jm
