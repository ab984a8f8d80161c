// Forwarding header: the B200 build declares the whole pipesim:: API in one
// place (pipesim_b200.hpp); this file keeps reference include paths working.
#ifndef PIPESIM_EXPORT_HPP_
#define PIPESIM_EXPORT_HPP_
#include "pipesim/pipesim_b200.hpp"
#endif
