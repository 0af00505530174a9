// Engine instantiation: Cartpole (dynamics.py:194-284) x CostCartpoleSwingup, float (one unit per
// (model, cost, precision): the units compile in parallel).
#include "engine.cuh"

namespace jm {
EngineBase* make_cartpole_swingup_f32() { return new Engine<Cartpole, CostCartpoleSwingup, float>(); }
}  // namespace jm
