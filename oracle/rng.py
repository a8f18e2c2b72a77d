"""SplitMix64 counter-based generator (TEST INFRASTRUCTURE -- see oracle/__init__.py).

Algorithm 1 draws random subsets and random great circles.
Both the oracle and the C++ order finder implement this same generator so that
the orders they produce can be compared bit for bit (BASELINE.json north_star:
"The order and slicing indices must be bit-identical").

  splitmix64(x): z = x + 0x9E3779B97F4A7C15; z = (z ^ z>>30) * 0xBF58476D1CE4E5B9;
                 z = (z ^ z>>27) * 0x94D049BB133111EB; return z ^ z>>31   (mod 2^64)
  stream(seed, sid): key = splitmix64(seed ^ splitmix64(sid)); draw i -> splitmix64(key + i)
  uniform: (u64 >> 11) * 2^-53  in [0, 1)
"""
M64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    z = (x + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def child_stream(sid: int, side: int) -> int:
    return splitmix64((sid * 2 + side + 1) & M64)


class Stream:
    def __init__(self, seed: int, sid: int):
        self.key = splitmix64((seed & M64) ^ splitmix64(sid & M64))
        self.ctr = 0

    def u64(self) -> int:
        v = splitmix64((self.key + self.ctr) & M64)
        self.ctr += 1
        return v

    def uniform(self) -> float:
        return float(self.u64() >> 11) * (1.0 / 9007199254740992.0)

    def below(self, m: int) -> int:
        return self.u64() % m
