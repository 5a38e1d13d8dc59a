"""B200-native A5/1 state-graph reduction, steps 1-3 (arXiv 1210.6411).

Drop-in for the reference package ``lfsrcycles`` on its hot path: the special-node
predicate, the leaf/predecessor filter, the step-1 enumeration, the step-2 prune, the
step-3 bitsliced chain walk and the edge records.  Batch work runs in hand-written
sm_100a kernels behind the C ABI of ``include/lfsr_b200.h``; there is no CPU fallback.
"""

from ._native import device_count, set_device  # noqa: F401  (fails loudly if the .so is missing)
from .bitslice import (DEFAULT_STRIDE_A51, SlicedBatch, StrideError, UnsupportedSpecError,  # noqa: F401
                       calibrate_stride, candidate_hops, clock_sliced, forward_to_candidate,
                       transpose, untranspose, walk_arrays)
from .cipher import (A51, CLOCK_PATTERNS, DEFAULT_FIXED_R3, MINI567, MINI789,  # noqa: F401
                     CandidateParams, CipherSpec, PredecessorTable, build_predecessor_table,
                     builtin_spec, clock_forward, default_fixed_r3, expected_chain_count,
                     expected_chain_length, is_candidate, majority_clock_mask,
                     minimum_cycle_length, parity_fold, predecessors, rank_state, shared_table,
                     step_register, table_index, unrank_state, unstep_register)
from .pipeline import (PruneConfig, PruneSoundnessError, PruneStats, auto_depth_limit,  # noqa: F401
                       build_skeleton_edges, enumerate_candidates, enumerate_candidates_array,
                       probe_segment, probe_segments, prune_shallow_segments, random_candidate,
                       random_candidates_gpu)
from .records import (EDGE_SIZE, ByteCounter, EdgeRecord, read_edge_arrays, read_edges,  # noqa: F401
                      read_states, write_edge_arrays, write_edges, write_states)
from .reduce import (CycleRecord, IterationLog, NotAPermutationError, PassStats,  # noqa: F401
                     ReduceConfig, count_cycles, count_cycles_arrays, cut_leaves_arrays,
                     cut_leaves_pass, cut_leaves_to_fixpoint, sort_edge_arrays)
from .ground_truth import CycleInfo, GroundTruth, brute_force_analysis  # noqa: F401
from .stats import (AnalysisReport, ExpectationTable, SampleStats, deviation_report,  # noqa: F401
                    random_mapping_expectations, sample_segment_distances, sample_segment_shapes)
from .step3 import merge_edge_files, walk_to_edge_files  # noqa: F401

__version__ = "0.1.0"
