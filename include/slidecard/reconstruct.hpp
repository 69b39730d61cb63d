// slidecard/reconstruct.hpp — B200 drop-in: the reconstruct types live in slidecard/window.hpp
// (proj/core/include/slidecard/reconstruct.hpp in the reference).
#pragma once

#include "slidecard/window.hpp"
