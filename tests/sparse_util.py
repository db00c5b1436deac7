"""Test-side readers of the PMS / CMS sparse cubes (decode, lookup with comparison count)."""
import bisect

import numpy as np

NONE = 0xFFFFFFFF


def decode(S, P, C, cms):
    out = np.zeros((P, C, 16), np.uint64)
    for q in range(S["n_planes"]):
        i0, i1 = int(S["index_off"][q]), int(S["index_off"][q + 1])
        assert S["index_id"][i1 - 1] == NONE                    # one sentinel closes the plane
        for i in range(i0, i1 - 1):
            b = int(S["index_id"][i])
            for v in range(int(S["index_start"][i]), int(S["index_start"][i + 1])):
                leaf = int(S["ids"][v])
                if cms:
                    out[leaf, q, b] = S["vals"][v]
                else:
                    out[q, b, leaf] = S["vals"][v]
    return out


def lookup(S, plane, inner, leaf):
    """(value or None, comparisons): binary search of the plane's sparse index, then of the
    leaf ids inside the segment."""
    i0, i1 = int(S["index_off"][plane]), int(S["index_off"][plane + 1]) - 1
    ids = [int(x) for x in S["index_id"][i0:i1]]
    comps = max(1, len(ids)).bit_length()
    k = bisect.bisect_left(ids, inner)
    if k == len(ids) or ids[k] != inner:
        return None, comps
    a, b = int(S["index_start"][i0 + k]), int(S["index_start"][i0 + k + 1])
    leaves = [int(x) for x in S["ids"][a:b]]
    comps += max(1, len(leaves)).bit_length()
    j = bisect.bisect_left(leaves, leaf)
    if j == len(leaves) or leaves[j] != leaf:
        return None, comps
    return int(S["vals"][a + j]), comps


def scan(S, plane, inner):
    i0, i1 = int(S["index_off"][plane]), int(S["index_off"][plane + 1]) - 1
    for i in range(i0, i1):
        if int(S["index_id"][i]) == inner:
            a, b = int(S["index_start"][i]), int(S["index_start"][i + 1])
            return [(int(S["ids"][v]), int(S["vals"][v])) for v in range(a, b)]
    return []
