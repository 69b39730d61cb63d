// slidecard/trace.hpp — B200 drop-in: the trace types live in slidecard/window.hpp
// (proj/core/include/slidecard/trace.hpp in the reference).
#pragma once

#include "slidecard/window.hpp"
