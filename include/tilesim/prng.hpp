// tilesim/prng.hpp -- the reference's header name, kept so translation units
// written against the reference include it unchanged.  Provides:
//   Prng: splitmix64-seeded xoshiro256**, the seed contract (proj/include/tilesim/prng.hpp)
// The declarations live in tilesim/core.hpp (the B200 build's gatecore, one
// header); the definitions are in libtilesim_b200.so.
#pragma once

#include "tilesim/core.hpp"
