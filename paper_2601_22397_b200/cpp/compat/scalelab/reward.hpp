// drop-in forwarder: reference callers include "scalelab/reward.hpp"
#pragma once
#include "scalelab_b200/reward.hpp"
