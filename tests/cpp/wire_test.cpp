// C++ host facade: wire codec + exception mapping (no GPU needed).
// Vectors from the reference's own tests (proj/tests/test_wire.cpp:32-150).
#include <cstdio>
#include <cstdlib>

#include "chunknet_b200.hpp"

using namespace chunknet::b200;

#define REQUIRE(x) do { if (!(x)) { std::fprintf(stderr, "FAILED %s:%d %s\n", __FILE__, __LINE__, #x); std::exit(1); } } while (0)

int main() {
    REQUIRE(encode_header({5, 3, 200, true, 0}) == 0x05079100u);
    REQUIRE(encode_header({255, 127, 255, true, 255}) == 0xFFFFFFFFu);
    REQUIRE((decode_header(0x05079100u) == ControlHeader{5, 3, 200, true, 0}));
    bool threw = false;
    try { encode_header({0, 128, 0, false, 0}); } catch (const FieldRangeError&) { threw = true; }
    REQUIRE(threw);
    REQUIRE(csn_before(254, 2, {250, 12}));
    REQUIRE(!csn_before(3, 252, {250, 12}));
    threw = false;
    try { csn_before(15, 12, {10, 5}); } catch (const OutOfWindowError&) { threw = true; }
    REQUIRE(threw);
    threw = false;
    try { csn_before(0, 0, {0, 129}); } catch (const FieldRangeError&) { threw = true; }
    REQUIRE(threw);
    for (unsigned w = 0; w < 200000; w += 7) REQUIRE(encode_header(decode_header(w * 2654435761u)) == w * 2654435761u);
    std::printf("CPP_WIRE_OK\n");
    return 0;
}
