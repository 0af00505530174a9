// Engine instantiation: Cartpole (dynamics.py:194-284) x CostDiagQuadratic, float (one unit per
// (model, cost, precision): the units compile in parallel).
#include "engine.cuh"

namespace jm {
EngineBase* make_cartpole_diag_f32() { return new Engine<Cartpole, CostDiagQuadratic, float>(); }
}  // namespace jm
