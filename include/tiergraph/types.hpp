// Forwarder: reference proj/include/tiergraph/types.hpp -> the B200 drop-in API.
#pragma once
#include "tiergraph/tiergraph.hpp"
