"""Independent pure-Python brute force.

A dense double loop over (query, key) with masked logits set to -inf, written
without numpy and without any code from oracle/.  Only for tiny inputs.
The mask is built here from the chunk lengths by its own loop.
"""
import math


def build_mask(chunk_lens):
    """mask[i][j] per P:137-143: key chunk in {0, c-1, c} of the query chunk."""
    owner = []
    for c, n in enumerate(chunk_lens):
        owner += [c] * n
    L = len(owner)
    mask = [[False] * L for _ in range(L)]
    for i in range(L):
        for j in range(L):
            ci, cj = owner[i], owner[j]
            mask[i][j] = (cj == 0) or (cj == ci) or (cj == ci - 1)
    return mask


def dense_masked_attention(q, k, v, mask, scale):
    """q, k, v: nested lists [L][H][d]; returns [L][H][d] as floats."""
    L = len(q)
    H = len(q[0])
    d = len(q[0][0])
    out = [[[0.0] * d for _ in range(H)] for _ in range(L)]
    for h in range(H):
        for i in range(L):
            logits = []
            for j in range(L):
                if mask[i][j]:
                    s = 0.0
                    for c in range(d):
                        s += q[i][h][c] * k[j][h][c]
                    logits.append(s * scale)
                else:
                    logits.append(-math.inf)
            mx = max(logits)
            w = [math.exp(x - mx) if x != -math.inf else 0.0 for x in logits]
            z = sum(w)
            for c in range(d):
                acc = 0.0
                for j in range(L):
                    acc += w[j] / z * v[j][h][c]
                out[i][h][c] = acc
    return out
