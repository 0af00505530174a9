// Engine instantiation: Cartpole (dynamics.py:194-284) x CostCartpoleSwingup, double (one unit per
// (model, cost, precision): the units compile in parallel).
#include "engine.cuh"

namespace jm {
EngineBase* make_cartpole_swingup_f64() { return new Engine<Cartpole, CostCartpoleSwingup, double>(); }
}  // namespace jm
