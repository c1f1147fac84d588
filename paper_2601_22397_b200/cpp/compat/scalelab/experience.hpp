// drop-in forwarder: reference callers include "scalelab/experience.hpp"
#pragma once
#include "scalelab_b200/experience.hpp"
