"""TEST-SIDE restatements of the reference h2.matvec (pkg/src/gcabem/h2.py:
49-71) and of the device product's staged algorithm on the descriptor
arrays that h2._leaf_arrays hands to the C ABI."""
import numpy as np


def matvec_reference(M, x):
    """Leaf loop in block-tree preorder, as h2.py:49-71."""
    rt, ct = M.block_tree.row_tree, M.block_tree.col_tree
    xp = np.asarray(x, dtype=np.complex128)[ct.permutation]
    yp = np.zeros(M.shape[0], dtype=np.complex128)
    for leaf in M.block_tree.leaves:
        t, s = rt.nodes[leaf.row], ct.nodes[leaf.col]
        xs = xp[s.start:s.start + s.size]
        P = M.payloads[leaf.index]
        if leaf.kind == "dense":
            yp[t.start:t.start + t.size] += P @ xs
        else:
            z = M.col_ops[leaf.col].V.T @ xs
            yp[t.start:t.start + t.size] += M.row_ops[leaf.row].V @ (P @ z)
    y = np.empty(M.shape[0], dtype=np.complex128)
    y[rt.permutation] = yp
    return y


def matvec_staged(M, x):
    """The device algorithm (csrc/h2_matvec.cu) on h2._leaf_arrays' tables."""
    from paper_1510_07244_b200 import h2
    desc, base, buf, (rdesc, nro), (cdesc, nco), V = h2._leaf_arrays(M)
    xp = np.asarray(x, dtype=np.complex128)[M.block_tree.col_tree.permutation]
    xs = [V[d[3]:d[3] + d[1] * d[2]].reshape(d[1], d[2]).T @ xp[d[0]:d[0] + d[1]]
          for d in cdesc[:nco]]
    z = [np.zeros(d[2], np.complex128) for d in rdesc[:nro]]
    yp = np.zeros(M.shape[0], dtype=np.complex128)
    for l in range(desc.shape[0]):
        r0, nr, c0, nc, dense, ro, co = desc[l]
        if dense:
            P = buf[base[l]:base[l] + nr * nc].reshape(nr, nc)
            yp[r0:r0 + nr] += P @ xp[c0:c0 + nc]
        else:
            kr, kc = rdesc[ro][2], cdesc[co][2]
            P = buf[base[l]:base[l] + kr * kc].reshape(kr, kc)
            z[ro] += P @ xs[co]
    for o in range(nro):
        s0, n, k, off = rdesc[o]
        yp[s0:s0 + n] += V[off:off + n * k].reshape(n, k) @ z[o]
    y = np.empty(M.shape[0], dtype=np.complex128)
    y[M.block_tree.row_tree.permutation] = yp
    return y
