#pragma once
// TEST INFRASTRUCTURE ONLY (built by oracle/Makefile into oracle/_ref/).
//
// Umbrella header for compiling the reference's UNMODIFIED acceptance suite
// (/root/reference/proj/tests/acceptance.cpp) against the drop-in codec.  The
// reference's own umbrella (proj/include/neuzip/neuzip.hpp:1-12) pulls in
// every header; here the codec headers resolve to this repo's include/neuzip/
// (include path order: this directory, repo include/, then the reference's
// include/), so compress/decompress run on the B200 through libnzgpu.so,
// while the headers the repo does not replace -- the reference's RNG, the
// CPU training harness that calls the codec per layer (nn.hpp:228-318) and
// the perturbation study -- come from the reference unchanged.
#include "neuzip/ans.hpp"
#include "neuzip/bitfloat.hpp"
#include "neuzip/crc32.hpp"
#include "neuzip/entropy.hpp"
#include "neuzip/errors.hpp"
#include "neuzip/nn.hpp"
#include "neuzip/parallel.hpp"
#include "neuzip/perturb.hpp"
#include "neuzip/rng.hpp"
#include "neuzip/tensorstore.hpp"
