// slidecard/report.hpp — B200 drop-in: the report types live in slidecard/window.hpp
// (proj/core/include/slidecard/report.hpp in the reference).
#pragma once

#include "slidecard/window.hpp"
