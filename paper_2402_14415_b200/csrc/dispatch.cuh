// Runtime (dim, order) -> template dispatch.
#pragma once

#define TGCU_DISPATCH(DIMV, ORDERV, ...)                                         \
    do {                                                                         \
        if ((DIMV) == 3) {                                                       \
            constexpr int DIM = 3;                                               \
            if ((ORDERV) == 2) { constexpr int ORDER = 2; __VA_ARGS__; }         \
            else if ((ORDERV) == 1) { constexpr int ORDER = 1; __VA_ARGS__; }    \
            else { constexpr int ORDER = 0; __VA_ARGS__; }                       \
        } else {                                                                 \
            constexpr int DIM = 2;                                               \
            if ((ORDERV) == 2) { constexpr int ORDER = 2; __VA_ARGS__; }         \
            else if ((ORDERV) == 1) { constexpr int ORDER = 1; __VA_ARGS__; }    \
            else { constexpr int ORDER = 0; __VA_ARGS__; }                       \
        }                                                                        \
    } while (0)

namespace tgcu {
inline int grid_blocks(long long n, int threads, int cap = 148 * 16) {
    long long b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > cap) b = cap;
    return (int)b;
}
}  // namespace tgcu
