"""ctypes binding of libivk.so (include/ivk.h).

The library is the ONLY compute path: if it is missing or fails to load,
every operator raises -- there is no CPU fallback.
"""

import ctypes as C
import os

__all__ = ["lib", "check", "OperatorDesc", "PatchDesc", "KronDesc", "TransferDesc", "CoarseDesc",
           "GeneralDesc", "GeneralTransferDesc", "ModalDesc",
           "IVK_MAX_STAGES", "IvkError", "SingularPatch"]

IVK_MAX_STAGES = 3
IVK_MAX_QUAD = 16
IVK_ESINGULAR = -3

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libivk.so")

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)
u8p = C.POINTER(C.c_uint8)


class IvkError(RuntimeError):
    pass


class SingularPatch(IvkError):
    pass


class K1Tiles(C.Structure):
    _fields_ = [
        ("n_tiles", C.c_int32), ("max_u", C.c_int32), ("max_p", C.c_int32),
        ("max_ent", C.c_int32), ("max_slices", C.c_int32), ("max_blob", C.c_int32),
        ("tile_rec", C.c_void_p), ("blob", C.c_void_p), ("ecol", C.c_void_p),
        ("eval", C.c_void_p),
    ]


class OperatorDesc(C.Structure):
    _fields_ = [
        ("stages", C.c_int32), ("n_nodes", C.c_int32), ("n_p", C.c_int32),
        ("n_conv", C.c_int32), ("nnz", C.c_int32), ("dt", C.c_double),
        ("butcher_a", C.c_double * (IVK_MAX_STAGES * IVK_MAX_STAGES)),
        ("p2_rowptr", C.c_void_p), ("p2_col", C.c_void_p), ("p2_mk", C.c_void_p),
        ("conv", C.c_void_p),
        ("b_rowptr", C.c_void_p), ("b_col", C.c_void_p), ("b_val", C.c_void_p),
        ("bt_rowptr", C.c_void_p), ("bt_col", C.c_void_p), ("bt_val", C.c_void_p),
        ("node_constrained", C.c_void_p),
        ("p2_sptr", C.c_void_p), ("p2_scol", C.c_void_p), ("p2_smk", C.c_void_p),
        ("conv_s", C.c_void_p), ("nnz_s", C.c_int32),
        ("b_sptr", C.c_void_p), ("b_scol", C.c_void_p), ("b_sval", C.c_void_p),
        ("bt_sptr", C.c_void_p), ("bt_scol", C.c_void_p), ("bt_sval", C.c_void_p),
        ("ncomp", C.c_int32),
        ("k1_tiles", C.POINTER(K1Tiles)),
        ("k1_order", C.c_void_p), ("k1_order_n", C.c_int32),
    ]


class KronDesc(C.Structure):
    _fields_ = [
        ("nblk", C.c_int32),
        ("is_complex", C.c_int32 * IVK_MAX_STAGES),
        ("lam_re", C.c_double * IVK_MAX_STAGES), ("lam_im", C.c_double * IVK_MAX_STAGES),
        ("v_re", C.c_double * (IVK_MAX_STAGES * IVK_MAX_STAGES)),
        ("v_im", C.c_double * (IVK_MAX_STAGES * IVK_MAX_STAGES)),
        ("vinv_re", C.c_double * (IVK_MAX_STAGES * IVK_MAX_STAGES)),
        ("vinv_im", C.c_double * (IVK_MAX_STAGES * IVK_MAX_STAGES)),
        ("scale", C.c_double * IVK_MAX_STAGES),
        ("symmetric", C.c_int32),
    ]


class ModalDesc(C.Structure):
    _fields_ = [
        ("stages", C.c_int32), ("ncomp", C.c_int32), ("dt", C.c_double),
        ("butcher_a", C.c_double * (IVK_MAX_STAGES * IVK_MAX_STAGES)),
        ("layout", C.c_int32),
    ]


class PatchDesc(C.Structure):
    _fields_ = [
        ("num_patches", C.c_int32), ("dim", C.c_int32), ("max_m", C.c_int32),
        ("total_m", C.c_int32),
        ("idx_off", C.c_void_p), ("idx", C.c_void_p), ("inv_off", C.c_void_p),
        ("inv", C.c_void_p), ("dof_ptr", C.c_void_p), ("dof_pos", C.c_void_p),
        ("vertex", C.c_void_p), ("node_off", C.c_void_p), ("node", C.c_void_p),
        ("slot_pos", C.c_void_p),
        ("kron", C.POINTER(KronDesc)),
        ("n_classes", C.c_int32),
        ("class_inv_off", C.c_void_p), ("class_inv", C.c_void_p),
        ("n_tiles", C.c_int32), ("tile_start", C.c_void_p), ("tile_class", C.c_void_p),
        ("tile_off", C.c_void_p), ("cidx", C.c_void_p), ("cdst", C.c_void_p),
        ("modal", C.POINTER(ModalDesc)),
    ]


class TransferDesc(C.Structure):
    _fields_ = [
        ("stages", C.c_int32), ("nf_nodes", C.c_int32), ("nf_p", C.c_int32),
        ("nc_nodes", C.c_int32), ("nc_p", C.c_int32),
        ("p2_rowptr", C.c_void_p), ("p2_col", C.c_void_p), ("p2_val", C.c_void_p),
        ("p2t_rowptr", C.c_void_p), ("p2t_col", C.c_void_p), ("p2t_val", C.c_void_p),
        ("p1_rowptr", C.c_void_p), ("p1_col", C.c_void_p), ("p1_val", C.c_void_p),
        ("p1t_rowptr", C.c_void_p), ("p1t_col", C.c_void_p), ("p1t_val", C.c_void_p),
        ("fine_constrained", C.c_void_p), ("coarse_constrained", C.c_void_p),
        ("ncomp", C.c_int32),
    ]


class CoarseDesc(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("nb", C.c_int32), ("l_ntiles", C.c_int32), ("u_ntiles", C.c_int32),
        ("stages", C.c_int32), ("n_u", C.c_int32), ("n_p", C.c_int32),
        ("l_colptr", C.c_void_p), ("l_row", C.c_void_p), ("l_tiles", C.c_void_p),
        ("l_diag", C.c_void_p),
        ("u_colptr", C.c_void_p), ("u_row", C.c_void_p), ("u_tiles", C.c_void_p),
        ("u_diag", C.c_void_p),
        ("perm_r", C.c_void_p), ("perm_c", C.c_void_p),
        ("dense", C.c_void_p), ("dense_ld", C.c_int32),
    ]


class PeerView(C.Structure):
    _fields_ = [("dof_ptr", C.c_void_p), ("dof_pos", C.c_void_p), ("local", C.c_void_p)]


class GeneralDesc(C.Structure):
    _fields_ = [
        ("stages", C.c_int32), ("n", C.c_int32), ("nnz", C.c_int32), ("dt", C.c_double),
        ("butcher_a", C.c_double * (IVK_MAX_STAGES * IVK_MAX_STAGES)),
        ("rowptr", C.c_void_p), ("col", C.c_void_p), ("ml", C.c_void_p),
        ("sptr", C.c_void_p), ("scol", C.c_void_p), ("sml", C.c_void_p),
        ("constrained", C.c_void_p),
    ]


class GeneralTransferDesc(C.Structure):
    _fields_ = [
        ("stages", C.c_int32), ("nf", C.c_int32), ("nc", C.c_int32),
        ("p_rowptr", C.c_void_p), ("p_col", C.c_void_p), ("p_val", C.c_void_p),
        ("pt_rowptr", C.c_void_p), ("pt_col", C.c_void_p), ("pt_val", C.c_void_p),
        ("fine_constrained", C.c_void_p), ("coarse_constrained", C.c_void_p),
    ]


class QuadTable(C.Structure):
    _fields_ = [
        ("nq", C.c_int32),
        ("w", C.c_double * IVK_MAX_QUAD),
        ("phi", C.c_double * (IVK_MAX_QUAD * 6)),
        ("dphi", C.c_double * (IVK_MAX_QUAD * 12)),
    ]


class ConvectionDesc(C.Structure):
    _fields_ = [
        ("n_cells", C.c_int32), ("n_nodes", C.c_int32), ("nnz", C.c_int32),
        ("quad", C.POINTER(QuadTable)),
        ("cell_nodes", C.c_void_p), ("cell_geo", C.c_void_p),
        ("entry_ptr", C.c_void_p), ("entry_contrib", C.c_void_p),
        ("row_of", C.c_void_p), ("col", C.c_void_p), ("node_constrained", C.c_void_p),
        ("sell_pos", C.c_void_p), ("node_ptr", C.c_void_p), ("node_contrib", C.c_void_p),
    ]


class MHDDesc(C.Structure):
    _fields_ = [
        ("n_cells", C.c_int32), ("nnz", C.c_int32), ("nq", C.c_int32),
        ("Re", C.c_double), ("Rm", C.c_double), ("S", C.c_double),
        ("w", C.c_double * IVK_MAX_QUAD),
        ("phi", C.c_double * (IVK_MAX_QUAD * 6)),
        ("dphi", C.c_double * (IVK_MAX_QUAD * 12)),
        ("psi", C.c_double * (IVK_MAX_QUAD * 3)),
        ("dpsi", C.c_double * 6),
        ("cell_geo", C.c_void_p), ("cell_nodes", C.c_void_p),
        ("entry_ptr", C.c_void_p), ("entry_contrib", C.c_void_p), ("sell_pos", C.c_void_p),
    ]


# name -> argtypes (restype int unless noted)
_P = C.c_void_p
_SIGS = {
    "ivk_last_error": ([], C.c_char_p),
    "ivk_version": ([], C.c_int),
    "ivk_launch_count": ([], C.c_int64),
    "ivk_stage_apply": ([C.POINTER(OperatorDesc), _P, _P, _P, _P], C.c_int),
    "ivk_patch_apply": ([C.POINTER(PatchDesc), _P, _P, _P], C.c_int),
    "ivk_patch_combine": ([C.POINTER(PatchDesc), _P, _P, C.c_double, C.c_double, _P, _P, _P, _P],
                          C.c_int),
    "ivk_patch_factor": ([C.POINTER(OperatorDesc), C.POINTER(PatchDesc), _P, _P], C.c_int),
    "ivk_stage_apply_slices": ([C.POINTER(OperatorDesc), _P, C.c_int32, _P, _P, _P, _P], C.c_int),
    "ivk_patch_combine_list": ([C.POINTER(PatchDesc), _P, C.c_int32, _P, _P, C.c_double,
                                C.c_double, _P, _P, _P, _P], C.c_int),
    "ivk_index_copy": ([C.c_int64, _P, _P, _P, _P, C.c_double, _P], C.c_int),
    "ivk_index_update": ([C.c_int64, _P, C.c_double, _P, C.c_double, _P, _P, _P, _P], C.c_int),
    "ivk_vanka_sweep": ([C.POINTER(OperatorDesc), C.POINTER(PatchDesc), _P, _P, C.c_double, _P,
                         _P, _P, _P, _P], C.c_int),
    "ivk_restrict": ([C.POINTER(TransferDesc), _P, _P, _P], C.c_int),
    "ivk_prolong_add": ([C.POINTER(TransferDesc), _P, _P, _P], C.c_int),
    "ivk_coarse_solve": ([C.POINTER(CoarseDesc), _P, _P, _P], C.c_int),
    "ivk_project_pressure_means": ([C.c_int32, C.c_int32, C.c_int32, _P, _P, _P], C.c_int),
    "ivk_axpby": ([C.c_int64, C.c_double, _P, C.c_double, _P, _P, _P], C.c_int),
    "ivk_seed_constrained": ([C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P, _P, _P, _P],
                             C.c_int),
    "ivk_convection_assemble": ([C.POINTER(ConvectionDesc), _P, _P, _P, _P, _P, _P], C.c_int),
    "ivk_reduction_scratch_bytes": ([], C.c_size_t),
    "ivk_dot": ([C.c_int64, _P, _P, _P, _P, _P], C.c_int),
    "ivk_norm": ([C.c_int64, _P, _P, _P, _P], C.c_int),
    "ivk_mgs": ([C.c_int64, _P, C.c_int64, C.c_int32, _P, _P, _P, _P, _P], C.c_int),
    "ivk_scale": ([C.c_int64, _P, _P, C.c_int32, _P, _P], C.c_int),
    "ivk_givens": ([C.c_int32, C.c_int32, _P, _P, _P, _P, _P, _P], C.c_int),
    "ivk_hessenberg_solve": ([C.c_int32, C.c_int32, _P, _P, _P, _P], C.c_int),
    "ivk_lincomb": ([C.c_int64, _P, C.c_int64, C.c_int32, _P, _P, _P], C.c_int),
    "ivk_patch_gather_blocks": ([C.POINTER(OperatorDesc), C.POINTER(PatchDesc), C.c_int32, _P,
                                 _P, _P, _P], C.c_int),
    "ivk_modal_factor": ([C.POINTER(PatchDesc), C.c_int32, _P, _P, _P, _P, _P], C.c_int),
    "ivk_peer_combine_update": ([C.c_int32, _P, _P, _P, _P, C.c_double, _P, _P, _P], C.c_int),
    "ivk_mhd_assemble": ([C.POINTER(MHDDesc), _P, _P, _P, _P, _P, _P], C.c_int),
    "ivk_general_apply": ([C.POINTER(GeneralDesc), _P, _P, _P, _P], C.c_int),
    "ivk_general_patch_factor": ([C.POINTER(GeneralDesc), C.POINTER(PatchDesc), _P, _P], C.c_int),
    "ivk_general_vanka_sweep": ([C.POINTER(GeneralDesc), C.POINTER(PatchDesc), _P, _P, C.c_double,
                                 _P, _P, _P, _P, _P], C.c_int),
    "ivk_general_seed_constrained": ([C.POINTER(GeneralDesc), _P, _P, _P], C.c_int),
    "ivk_general_restrict": ([C.POINTER(GeneralTransferDesc), _P, _P, _P], C.c_int),
    "ivk_general_prolong_add": ([C.POINTER(GeneralTransferDesc), _P, _P, _P], C.c_int),
}
EXPORTED = tuple(_SIGS)

_lib = None


def load(path=_LIB_PATH):
    """Load libivk.so (raises if it is absent -- no fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise IvkError(
            f"libivk.so not found at {path}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
    lib = C.CDLL(path)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def lib():
    return load()


PROJECT_BLOCKS = 64   # IVK_PROJECT_BLOCKS (include/ivk.h)


def reduction_scratch():
    """A fresh zeroed device scratch for ivk_dot / ivk_norm / ivk_mgs (one
    per concurrent stream of reductions; include/ivk.h)."""
    import torch
    from ._device import device
    nbytes = int(lib().ivk_reduction_scratch_bytes())
    return torch.zeros((nbytes + 7) // 8, dtype=torch.float64, device=device())


def check(rc, what=""):
    if rc == 0:
        return
    msg = load().ivk_last_error().decode(errors="replace")
    if rc == IVK_ESINGULAR:
        raise SingularPatch(f"{what}: {msg}")
    raise IvkError(f"{what} failed ({rc}): {msg}")
