// Engine instantiation: Quadrotor (dynamics.py:296-409) x CostDiagQuadratic, float (one unit per
// (model, cost, precision): the units compile in parallel).
#include "engine.cuh"

namespace jm {
EngineBase* make_quadrotor_diag_f32() { return new Engine<Quadrotor, CostDiagQuadratic, float>(); }
}  // namespace jm
