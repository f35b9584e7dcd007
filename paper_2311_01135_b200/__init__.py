"""B200-native batched restricted-KS B3LYP/STO-3G label generator.

Drop-in for the reference SCF driver path (deskdft): `scf`, `properties`,
`SCFOptions`, `SCFResult`, `Molecule`, `load_basis`, `expand`, ... plus the
batched `scf_batch` and the labeling pipeline (`paper_2311_01135_b200.pipeline`:
JSONL records, checkpoint/resume, several device batches in flight).  All compute runs in libqm1b_b200.so (sm_100a CUDA) through
the C ABI in include/qm1b_b200.h.
"""

__version__ = "0.1.0"

from .basis import AOBasis, BasisSet, ContractedShell, expand, load_basis  # noqa: F401
from .errors import (BasisError, DeskDFTError, DeviceError, DimensionError,  # noqa: F401
                     MoleculeError, ResourceLimitError, XYZParseError)
from .molio import (GeometryManifest, ManifestEntry, Molecule, electron_count, emit_xyz,  # noqa: F401
                    load_manifest, nuclear_repulsion, parse_xyz, save_manifest)
from .scf import (OrbitalSolution, SCFOptions, SCFResult, diis_step, properties, scf,  # noqa: F401
                  scf_batch, scf_batch_device, solve_roothaan)
