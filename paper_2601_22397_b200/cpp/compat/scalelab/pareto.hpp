// drop-in forwarder: reference callers include "scalelab/pareto.hpp"
#pragma once
#include "scalelab_b200/pareto.hpp"
