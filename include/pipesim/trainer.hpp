// Forwarding header: the B200 build declares the whole pipesim:: API in one
// place (pipesim_b200.hpp); this file keeps reference include paths working.
#ifndef PIPESIM_TRAINER_HPP_
#define PIPESIM_TRAINER_HPP_
#include "pipesim/pipesim_b200.hpp"
#endif
