"""Independent pin for S -> S S | a (SURVEY V-5): R_S = the strict transitive closure of the
a-edges, {(i, j) : a path of >= 1 edges leads from i to j}.  Textbook construction, no CFPQ
arithmetic: strongly connected components (scipy), the condensation DAG in reverse
topological order, reach[c] = OR of (members(d) | reach[d]) over the successors d of c; a
node of a cyclic component (size > 1 or a self-loop) also reaches every member of its own.
Rows come back as uint32 bit rows in the library's layout (bit j of row i = word j >> 5,
bit j & 31), so whole matrices compare bit for bit."""
import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components


def strict_closure_bits(n, src, dst):
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    W = (n + 63) // 64
    A = sp.csr_matrix((np.ones(len(src), np.int8), (src, dst)), shape=(n, n))
    nc, lab = connected_components(A, directed=True, connection="strong")
    members = [[] for _ in range(nc)]
    for v in range(n):
        members[lab[v]].append(v)
    size = np.bincount(lab, minlength=nc)
    cyclic = size > 1
    loops = src[src == dst]
    cyclic[lab[loops]] = True
    # condensation edges
    cs, cd = lab[src], lab[dst]
    keep = cs != cd
    pairs = np.unique(np.stack([cs[keep], cd[keep]], 1), axis=0) if keep.any() else np.zeros((0, 2), np.int64)
    succ = [[] for _ in range(nc)]
    indeg = np.zeros(nc, np.int64)
    for a, b in pairs.tolist():
        succ[a].append(b)
        indeg[b] += 1
    order = [c for c in range(nc) if indeg[c] == 0]
    k = 0
    while k < len(order):
        for d in succ[order[k]]:
            indeg[d] -= 1
            if indeg[d] == 0:
                order.append(d)
        k += 1
    assert len(order) == nc
    mem_bits = np.zeros((nc, W), np.uint64)
    for c in range(nc):
        m = np.asarray(members[c])
        np.bitwise_or.at(mem_bits[c], m >> 6, (np.uint64(1) << (m & 63).astype(np.uint64)))
    reach = np.zeros((nc, W), np.uint64)
    for c in reversed(order):
        acc = reach[c]
        for d in succ[c]:
            acc |= mem_bits[d]
            acc |= reach[d]
    rows = np.zeros((n, W), np.uint64)
    for c in range(nc):
        row = reach[c] | (mem_bits[c] if cyclic[c] else np.uint64(0))
        rows[members[c]] = row
    # uint64 little-endian rows -> uint32 words of the library layout
    return rows.view(np.uint32).reshape(n, 2 * W)[:, : (n + 31) // 32]
