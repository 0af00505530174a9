// Engine instantiation: Quadrotor (dynamics.py:296-409) x CostQuadrotorHover, float (one unit per
// (model, cost, precision): the units compile in parallel).
#include "engine.cuh"

namespace jm {
EngineBase* make_quadrotor_hover_f32() { return new Engine<Quadrotor, CostQuadrotorHover, float>(); }
}  // namespace jm
