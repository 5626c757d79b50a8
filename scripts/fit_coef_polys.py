"""Offline fit of the fp64 coefficient polynomials (csrc/device_fp.cuh):
sin(pi r) = r P(r^2) on |r| <= 1/2 (near-minimax via Chebyshev interpolation in mpmath),
and the 2^(j/32) double-double table + degree-6 Taylor for exp on |r| <= ln2/64."""
import mpmath as mp
mp.mp.dps = 60
def fit_sinpi(n):
    f = lambda s: mp.sin(mp.pi * mp.sqrt(s)) / mp.sqrt(s) if s > 0 else mp.pi
    poly, err = mp.chebyfit(f, [0, mp.mpf(1) / 4], n, error=True)
    return poly[::-1], err  # ascending powers of s
if __name__ == "__main__":
    for n in (10, 11, 12, 13):
        c, e = fit_sinpi(n)
        print(n, "terms, abs err on P", mp.nstr(e, 5), " rel ~", mp.nstr(e / mp.pi, 5), " 2^-53 =", mp.nstr(mp.mpf(2) ** -53, 5))
    c, e = fit_sinpi(11)
    print("SINPI11 = {" + ", ".join(repr(float(x)) for x in c) + "}")
    hi = [float(mp.mpf(2) ** (mp.mpf(j) / 32)) for j in range(32)]
    lo = [float(mp.mpf(2) ** (mp.mpf(j) / 32) - mp.mpf(h)) for j, h in zip(range(32), hi)]
    print("EXP2_HI = {" + ", ".join(repr(x) for x in hi) + "}")
    print("EXP2_LO = {" + ", ".join(repr(x) for x in lo) + "}")
    l = mp.log(2) / 32
    lhi = float(l); 
    # Cody-Waite split with lhi having trailing zeros so n * lhi is exact for |n| < 2^15
    import struct
    b = struct.unpack("<Q", struct.pack("<d", float(l)))[0] & ~((1 << 20) - 1)
    lhi = struct.unpack("<d", struct.pack("<Q", b))[0]
    llo = float(l - mp.mpf(lhi))
    print("LN2_32_HI =", repr(lhi), " LN2_32_LO =", repr(llo), " INV =", repr(float(32 / mp.log(2))))
