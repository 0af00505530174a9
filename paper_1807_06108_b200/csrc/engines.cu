// Plugin -> engine dispatch (jm_create): one Engine<Dyn, Cost, Real> per
// (model, cost, precision), each instantiated in its own sys_*.cu unit.
#include "internal.h"

namespace jm {
EngineBase* make_cartpole_swingup_f32();
EngineBase* make_cartpole_swingup_f64();
EngineBase* make_cartpole_diag_f32();
EngineBase* make_cartpole_diag_f64();
EngineBase* make_quadrotor_hover_f32();
EngineBase* make_quadrotor_hover_f64();
EngineBase* make_quadrotor_diag_f32();
EngineBase* make_quadrotor_diag_f64();
EngineBase* make_linear_2x1_f32();
EngineBase* make_linear_2x1_f64();
EngineBase* make_linear_4x1_f32();
EngineBase* make_linear_4x1_f64();
EngineBase* make_linear_4x2_f32();
EngineBase* make_linear_4x2_f64();
EngineBase* make_linear_6x3_f32();
EngineBase* make_linear_6x3_f64();

// CartpoleModel (dynamics.py:194-284) with CartpoleStateCost or the diagonal quadratic cost
EngineBase* make_engine_cartpole(int cost_kind, int precision) {
  const bool f64 = precision == JM_F64;
  if (cost_kind == JM_COST_CARTPOLE_SWINGUP) return f64 ? make_cartpole_swingup_f64() : make_cartpole_swingup_f32();
  if (cost_kind == JM_COST_DIAG_QUADRATIC) return f64 ? make_cartpole_diag_f64() : make_cartpole_diag_f32();
  return nullptr;
}

// QuadrotorModel (dynamics.py:296-409) with QuadrotorStateCost or the diagonal quadratic cost
EngineBase* make_engine_quadrotor(int cost_kind, int precision) {
  const bool f64 = precision == JM_F64;
  if (cost_kind == JM_COST_QUADROTOR_HOVER) return f64 ? make_quadrotor_hover_f64() : make_quadrotor_hover_f32();
  if (cost_kind == JM_COST_DIAG_QUADRATIC) return f64 ? make_quadrotor_diag_f64() : make_quadrotor_diag_f32();
  return nullptr;
}

// the generic linear plugin, (n, m) in {(2,1), (4,1), (4,2), (6,3)}
EngineBase* make_engine_linear(int cost_kind, int precision, int n, int m) {
  if (cost_kind != JM_COST_DIAG_QUADRATIC) return nullptr;
  const bool f64 = precision == JM_F64;
  if (n == 2 && m == 1) return f64 ? make_linear_2x1_f64() : make_linear_2x1_f32();
  if (n == 4 && m == 1) return f64 ? make_linear_4x1_f64() : make_linear_4x1_f32();
  if (n == 4 && m == 2) return f64 ? make_linear_4x2_f64() : make_linear_4x2_f32();
  if (n == 6 && m == 3) return f64 ? make_linear_6x3_f64() : make_linear_6x3_f32();
  return nullptr;
}
}  // namespace jm
