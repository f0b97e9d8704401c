// carve/carve.hpp — umbrella header (drop-in for the reference's carve.hpp).
#pragma once
#include "carve/bench.hpp"
#include "carve/carver.hpp"
#include "carve/energy.hpp"
#include "carve/error.hpp"
#include "carve/raster.hpp"
#include "carve/solvers.hpp"
