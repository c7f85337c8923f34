// Forwarder: reference proj/include/tiergraph/csr_graph.hpp -> the B200 drop-in API.
#pragma once
#include "tiergraph/tiergraph.hpp"
