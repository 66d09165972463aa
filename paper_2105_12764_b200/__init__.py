"""B200-native multigrid data refactoring (arXiv 2105.12764).

The hot path -- MGARD-style multilevel decompose / recompose of structured
1-D/2-D/3-D grids -- runs in hand-written sm_100a kernels (csrc/) behind the
C ABI include/mgrg.h.  This package is the host-side mirror of the
reference's C++ API (refactor.py), the device-level plan handle (plan.py) and
the multi-GPU block driver (parallel.py)."""
from . import errors
from .errors import (CorruptFile, Error, InvalidBound, InvalidFusion, InvalidGrid,
                     InvalidLevel, IoError, MissingClass, ShapeError, SingularSystem,
                     TooManyWorkers, WorkerFailure)
from .plan import Plan
from .coop import (CommReport, CoopOptions, Partition, PartitionScheme,
                   cooperative_decompose, grouped_decompose, make_partitions,
                   split_dims_of)
from .container import (CompressionReport, CompressResult, DecompressResult, ReadResult,
                        RefactorFileHeader, compress, crc32, decompress, read_refactored,
                        read_refactored_header, write_refactored)
from .refactor import (LevelPassStats, PassStats, PhaseCounters, ReconstructionReport,
                       RefactoredData, RefactorOptions, TensorGrid, decompose,
                       decompose_spatiotemporal, make_grid,
                       recompose, recompose_with_report, uniform_coords, value_range,
                       weighted_l2_norm)
from .parallel import (BlockShardedRefactor, embarrassing_decompose, embarrassing_recompose,
                       split_blocks)

__all__ = [
    "Plan", "TensorGrid", "RefactoredData", "RefactorOptions", "PassStats",
    "LevelPassStats", "PhaseCounters", "ReconstructionReport", "decompose", "recompose",
    "decompose_spatiotemporal", "cooperative_decompose", "CoopOptions", "CommReport",
    "PartitionScheme", "Partition", "make_partitions", "split_dims_of", "grouped_decompose",
    "recompose_with_report", "make_grid", "uniform_coords", "value_range",
    "weighted_l2_norm", "errors", "Error", "InvalidGrid", "InvalidLevel", "ShapeError",
    "InvalidFusion", "SingularSystem", "TooManyWorkers", "WorkerFailure", "CorruptFile",
    "MissingClass", "InvalidBound", "IoError", "embarrassing_decompose",
    "embarrassing_recompose", "BlockShardedRefactor", "split_blocks", "crc32",
    "write_refactored", "read_refactored", "read_refactored_header", "ReadResult",
    "RefactorFileHeader", "compress", "decompress", "CompressResult", "DecompressResult",
    "CompressionReport",
]
