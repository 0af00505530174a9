// Engine instantiations for QuadrotorModel (dynamics.py:296-409).
#include "engine.cuh"

namespace jm {
EngineBase* make_engine_quadrotor(int cost_kind, int precision) {
  const bool f64 = precision == JM_F64;
  switch (cost_kind) {
    case JM_COST_QUADROTOR_HOVER:
      if (f64) return new Engine<Quadrotor, CostQuadrotorHover, double>();
      return new Engine<Quadrotor, CostQuadrotorHover, float>();
    case JM_COST_DIAG_QUADRATIC:
      if (f64) return new Engine<Quadrotor, CostDiagQuadratic, double>();
      return new Engine<Quadrotor, CostDiagQuadratic, float>();
    default:
      return nullptr;
  }
}
}  // namespace jm
