import mpmath, struct
mpmath.mp.prec = 200
N=128
def d2u(x): return struct.unpack('<Q', struct.pack('<d', x))[0]
out=[]
for k in range(N):
    e = mpmath.power(2, mpmath.mpf(k)/N)
    H = float(e)  # round to nearest double
    T = float(e/mpmath.mpf(H) - 1)
    out.append(d2u(T)); out.append((d2u(H) - ((k << 52)//N)) & 0xffffffffffffffff)
print(",\n".join("0x%016xULL"%v for v in out))
