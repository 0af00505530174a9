// Engine instantiations for CartpoleModel (dynamics.py:194-284).
#include "engine.cuh"

namespace jm {
EngineBase* make_engine_cartpole(int cost_kind, int precision) {
  const bool f64 = precision == JM_F64;
  switch (cost_kind) {
    case JM_COST_CARTPOLE_SWINGUP:
      if (f64) return new Engine<Cartpole, CostCartpoleSwingup, double>();
      return new Engine<Cartpole, CostCartpoleSwingup, float>();
    case JM_COST_DIAG_QUADRATIC:
      if (f64) return new Engine<Cartpole, CostDiagQuadratic, double>();
      return new Engine<Cartpole, CostDiagQuadratic, float>();
    default:
      return nullptr;
  }
}
}  // namespace jm
