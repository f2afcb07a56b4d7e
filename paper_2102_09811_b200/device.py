"""Device-resident mesh and quadrature tables (host precompute -> HBM).

Everything the reference builds on the host before its pass loop
(heatbem/assembly.py:201-206: vertex arrays, both product rules, the
touching CSR with case ids and permutations, the Duffy tables) is built
here with numpy once per (mesh, quadrature config) and uploaded as
contiguous float64 / int64 tensors.  Three index lists are added for the
device work decomposition: the singular work list (touching CSR positions
per test row, upper-triangular for symmetric operators), the node stars
(element, local vertex) per node for the p1 gathers, and the per-triangle
surface curls of the hat functions (heatbem/assembly.py:289-311).
"""
from __future__ import annotations

import weakref

import numpy as np

from . import _native
from .quadrature import QuadratureConfig, duffy_tables, rule_tables, touching_csr


def _curls(mesh) -> np.ndarray:
    """curl of hat i on triangle e = (v_{i+1} - v_{i+2}) / (2 area_e): (E_x, 3, 3)."""
    v = mesh.triangle_vertices()
    out = np.empty((mesh.n_triangles, 3, 3))
    for i in range(3):
        out[:, i, :] = (v[:, (i + 1) % 3, :] - v[:, (i + 2) % 3, :]) / (2.0 * mesh.areas[:, None])
    return out


class HostTables:
    """numpy side of the device tables (also what the CPU oracle consumes)."""

    def __init__(self, mesh, config: QuadratureConfig):
        c = np.ascontiguousarray
        self.E_x, self.N_x = mesh.n_triangles, mesh.n_vertices
        self.tri_nodes = c(mesh.triangles, dtype=np.int64)
        self.verts_tri = c(mesh.triangle_vertices())
        self.normals, self.centroids = c(mesh.normals), c(mesh.centroids)
        self.diameters, self.areas = c(mesh.diameters), c(mesh.areas)
        self.reg = [c(a) for a in rule_tables(mesh, config.regular_order)]
        self.near = [c(a) for a in rule_tables(mesh, config.near_order)]
        self.tn = [c(a) for a in touching_csr(mesh)]
        self.duf = [c(a) for a in duffy_tables(config.singular_order)]
        indptr, idx = self.tn[0], self.tn[1]
        rows = np.repeat(np.arange(self.E_x, dtype=np.int64), np.diff(indptr))
        self.sing_row = rows
        self.sing = {}
        for sym in (False, True):
            keep = idx >= rows if sym else np.ones(len(idx), dtype=bool)
            pos = np.flatnonzero(keep).astype(np.int64)
            cnt = np.bincount(rows[keep], minlength=self.E_x)
            rp = np.zeros(self.E_x + 1, dtype=np.int64)
            np.cumsum(cnt, out=rp[1:])
            self.sing[sym] = (pos, rp, int(cnt.max()) if len(cnt) else 0)
        self.star = [c(a) for a in mesh.node_star()]
        self.star_max = int(np.diff(self.star[0]).max())
        self.curls = c(_curls(mesh))
        self.curl_plan = curl_tile_plan(self.star[0], self.star[1], self.N_x)


CURL_TILE = 32   # nodes per tile of the curl-combine kernel (hb_capi.cu kCT)


def curl_tile_plan(star_indptr, star_elem, n_nodes: int, tile: int = CURL_TILE):
    """Per 32-node tile the sorted distinct elements of its node stars
    (eptr, elem) and, per star entry, its position in its tile's list
    (int32), plus the max list length and max star entries per tile."""
    nt = -(-n_nodes // tile)
    eptr = np.zeros(nt + 1, dtype=np.int64)
    pos = np.empty(len(star_elem), dtype=np.int32)
    lists, smax = [], 0
    for t in range(nt):
        s0, s1 = int(star_indptr[tile * t]), int(star_indptr[min(n_nodes, tile * t + tile)])
        u = np.unique(star_elem[s0:s1])
        lists.append(u)
        eptr[t + 1] = eptr[t] + len(u)
        pos[s0:s1] = np.searchsorted(u, star_elem[s0:s1])
        smax = max(smax, s1 - s0)
    elem = np.concatenate(lists).astype(np.int64) if lists else np.zeros(0, np.int64)
    return eptr, elem, pos, int(np.diff(eptr).max()) if nt else 0, int(smax)


class _LazyViews:
    """``tables.t[name]``: the device view of one table, made on first use."""

    def __init__(self, owner):
        self._o, self._v = owner, {}

    def __getitem__(self, name):
        v = self._v.get(name)
        if v is None:
            o = self._o
            off, n, dt, shape = o._where[id(o._names[name])]
            v = self._v[name] = o._blob[off:off + n].view(dt).view(shape)
        return v

    def __contains__(self, name):
        return name in self._o._names


class DeviceTables:
    """Device copies of :class:`HostTables` plus ready-made C descriptors.
    With ``pinned`` host staging the uploads are async copies from page-locked
    memory (the end-to-end benchmark path)."""

    def __init__(self, mesh, config: QuadratureConfig, device, host: HostTables | None = None):
        import torch

        self.host = H = host if host is not None else host_tables(mesh, config)
        self.device = device
        # every array in one buffer: one allocation and one host->device copy
        # (asynchronous from the page-locked blob of pin_host_tables)
        blob, where = _packed(H)
        self._blob = blob.to(device, non_blocking=True)

        # name -> host array; device views are made on first use (``t[name]``),
        # the descriptors take base + offset directly (no per-table tensor ops
        # on the upload path: the cold-table call stays one async copy)
        self._where = where
        self._names = {
            "tri_nodes": H.tri_nodes, "verts_tri": H.verts_tri, "normals": H.normals,
            "centroids": H.centroids, "diameters": H.diameters, "areas": H.areas,
            "reg_hats": H.reg[0], "reg_w": H.reg[1], "reg_pts": H.reg[2],
            "near_hats": H.near[0], "near_w": H.near[1], "near_pts": H.near[2],
            "tn_indptr": H.tn[0], "tn_idx": H.tn[1], "tn_case": H.tn[2],
            "tn_permt": H.tn[3], "tn_perms": H.tn[4],
            "duf_off": H.duf[0], "duf_t": H.duf[1], "duf_s": H.duf[2], "duf_w": H.duf[3],
            "sing_row": H.sing_row,
            "star_indptr": H.star[0], "star_elem": H.star[1], "star_local": H.star[2],
            "curls": H.curls,
            "curl_tile_eptr": H.curl_plan[0], "curl_tile_elem": H.curl_plan[1],
            "curl_star_pos": H.curl_plan[2],
        }
        for sym in (False, True):
            pos, rp, _ = H.sing[sym]
            self._names[f"sing_pos_{int(sym)}"] = pos
            self._names[f"sing_rowptr_{int(sym)}"] = rp
        self.t = _LazyViews(self)
        self._desc = {sym: self._make_desc(sym) for sym in (False, True)}

    def _make_desc(self, symmetric: bool) -> _native.MeshDesc:
        H = self.host
        base, where, t = self._blob.data_ptr(), self._where, self._names

        def p(a):   # device address of a table: blob base + its section offset
            return base + where[id(a)][0]
        d = _native.MeshDesc()
        d.E_x, d.N_x = H.E_x, H.N_x
        d.tri_nodes_dev, d.verts_tri_dev = p(t["tri_nodes"]), p(t["verts_tri"])
        d.normals_dev, d.centroids_dev = p(t["normals"]), p(t["centroids"])
        d.diameters_dev, d.areas_dev = p(t["diameters"]), p(t["areas"])
        d.reg_hats_dev, d.reg_w_dev, d.reg_pts_dev = p(t["reg_hats"]), p(t["reg_w"]), p(t["reg_pts"])
        d.n_reg = len(H.reg[1])
        d.near_hats_dev, d.near_w_dev, d.near_pts_dev = p(t["near_hats"]), p(t["near_w"]), p(t["near_pts"])
        d.n_near = len(H.near[1])
        d.tn_indptr_dev, d.tn_idx_dev, d.tn_case_dev = p(t["tn_indptr"]), p(t["tn_idx"]), p(t["tn_case"])
        d.tn_permt_dev, d.tn_perms_dev = p(t["tn_permt"]), p(t["tn_perms"])
        d.duf_off_dev, d.duf_t_dev = p(t["duf_off"]), p(t["duf_t"])
        d.duf_s_dev, d.duf_w_dev = p(t["duf_s"]), p(t["duf_w"])
        s = int(symmetric)
        d.sing_pos_dev, d.sing_rowptr_dev = p(t[f"sing_pos_{s}"]), p(t[f"sing_rowptr_{s}"])
        d.sing_max_per_row = H.sing[symmetric][2]
        d.sing_row_dev = p(t["sing_row"])
        d.star_indptr_dev, d.star_elem_dev = p(t["star_indptr"]), p(t["star_elem"])
        d.star_local_dev = p(t["star_local"])
        d.star_max = H.star_max
        d.curl_tile_eptr_dev, d.curl_tile_elem_dev = p(t["curl_tile_eptr"]), p(t["curl_tile_elem"])
        d.curl_star_pos_dev = p(t["curl_star_pos"])
        d.curl_tile_emax, d.curl_tile_smax = H.curl_plan[3], H.curl_plan[4]
        return d

    def desc(self, symmetric: bool) -> _native.MeshDesc:
        return self._desc[bool(symmetric)]


_CACHE: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()
_HOST: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def host_tables(mesh, config: QuadratureConfig) -> HostTables:
    per_mesh = _HOST.setdefault(mesh, {})
    key = (config.regular_order, config.singular_order)
    if key not in per_mesh:
        per_mesh[key] = HostTables(mesh, config)
    return per_mesh[key]


def _table_arrays(H: HostTables) -> list:
    arrays = [H.tri_nodes, H.verts_tri, H.normals, H.centroids, H.diameters, H.areas, *H.reg, *H.near,
              *H.tn, *H.duf, H.sing_row, *H.star, H.curls, *H.curl_plan[:3]]
    for sym in (False, True):
        arrays += list(H.sing[sym][:2])
    return arrays


def _packed(H: HostTables):
    """The host tables as one byte blob (256-byte aligned sections) and, per
    array id, (offset, bytes, torch dtype, shape); cached on ``H`` (the
    page-locked blob of pin_host_tables when pinned)."""
    import torch

    if getattr(H, "_blob", None) is None:
        arrays = _table_arrays(H)
        where, off = {}, 0
        for a in arrays:   # keyed by the attribute objects DeviceTables looks up
            where[id(a)] = (off, a.nbytes, torch.from_numpy(np.ascontiguousarray(a[:0])).dtype, tuple(a.shape))
            off += -(-a.nbytes // 256) * 256
        blob = np.zeros(max(off, 256), dtype=np.uint8)
        for a in arrays:
            o, n, _, _ = where[id(a)]
            blob[o:o + n] = np.ascontiguousarray(a).reshape(-1).view(np.uint8)
        H._blob, H._where = torch.from_numpy(blob), where
    return H._blob, H._where


def pin_host_tables(H: HostTables):
    """Page-locked copy of the packed host tables (the upload becomes one
    async DMA)."""
    blob, _ = _packed(H)
    if not blob.is_pinned():
        H._blob = blob.pin_memory()
    H.pinned_bytes = H._blob.numel()
    return H


def drop_device_tables(mesh):
    """Forget the uploaded tables of a mesh (next call re-uploads them)."""
    _CACHE.pop(mesh, None)


def device_tables(mesh, config: QuadratureConfig, device=None) -> DeviceTables:
    """Cached per mesh object (meshes are treated as immutable, as in the
    reference), quadrature config and device."""
    import torch

    _native.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    per_mesh = _CACHE.setdefault(mesh, {})
    key = (config.regular_order, config.singular_order, str(dev))
    if key not in per_mesh:
        per_mesh[key] = DeviceTables(mesh, config, dev, host_tables(mesh, config))
    return per_mesh[key]
