"""B200-native PSCA activity-detection hot path (arXiv 2503.15259).

Drop-in for the solver API of the reference package ``actdet``
(/root/reference/pkg/src/actdet/__init__.py:12-24): the same names, argument
meanings and error behaviour, with the PSCA iteration running as hand-written
sm_100a CUDA kernels behind the C ABI in include/psca.h.  Batched entry
points (``psca_run_batch``, ``unroll.forward_batch``) are the throughput path;
``harness`` runs the reference's experiment grid on GPU batches and
``unroll.train`` tunes PSCA-Nets with batched device forwards;
``baselines.pg_ml_batch`` is the projected-gradient comparison detector.
"""

from .sysmodel import (ActivityModel, DomainError, Sample, SystemConfig, empirical_cov,
                       gen_dataset, normalize_noise, sample_scene)
from .estimators import (DetectorTrace, Problem, StepSchedule, psca_run, psca_run_batch,
                         psca_run_batch_host,
                         default_schedule, default_steps, bounds_for)
from .priors import EffPathlossPrior, IndependentPrior, PairwiseMvbPrior
from .covlinalg import (ConditioningError, CovState, cov_known, cov_unknown, eval_objective,
                        frobenius_inverse, quad_forms)

__all__ = [
    "ActivityModel", "DomainError", "Sample", "SystemConfig", "empirical_cov",
    "gen_dataset", "normalize_noise", "sample_scene",
    "DetectorTrace", "Problem", "StepSchedule", "psca_run", "psca_run_batch", "psca_run_batch_host",
    "default_schedule", "default_steps", "bounds_for",
    "EffPathlossPrior", "IndependentPrior", "PairwiseMvbPrior",
    "ConditioningError", "CovState", "cov_known", "cov_unknown", "eval_objective",
    "frobenius_inverse", "quad_forms",
]
