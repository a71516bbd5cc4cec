"""The drop-in seams of the reference CLI's batched commands.

The reference's ``cmd_rank`` evaluates every schedule through
``es_mod.evaluate_population(schedules, evaluate, jobs=args.jobs, errors=errors)``
(ls/cli.py:115-121) and ``cmd_search`` calls ``es_mod.optimize(...)``
(ls/cli.py:152).  A loopscout maintainer switches both commands to the device
by replacing those two calls:

    results = backend.evaluate_schedules(program, schedules, arch, launch, jobs=args.jobs, errors=errors)
    result = backend.optimize(program, space, arch, params, jobs=args.jobs, launch=launch)

and ``cmd_analyze --code`` (ls/cli.py:89) calls ``backend.extract_features(program, code, arch,
launch, diagnostics)``: the user's assembly / PTX parsed on the device (code.py, csrc/code.cu).

Everything else in the reference CLI (report assembly, sorting, printing, exit
codes) stays as it is.  Both functions accept the reference's own objects
(LoopProgram, Schedule, ArchSpec, KernelLaunch, EsParams) as well as this
package's mirrors.
"""

from __future__ import annotations

from . import abi
from .arch import CostModelError
from .cost import score_batch
from .es import optimize as _optimize
from .ir import ProgramError, failure_message


def _exception(program, schedule, res, i: int) -> Exception:
    """The exception the reference's per-candidate closure raises for a failed candidate: the
    ProgramError text rebuilt from the schedule (ls/ir.py:151, 361-470), a host-side
    CostModelError (ls/cost.py:137-138), else the device status."""
    if i in res.messages and res.messages[i][0] == "CostModelError":
        return CostModelError(res.messages[i][1])
    msg = failure_message(program, schedule)
    if msg is not None:
        return ProgramError(msg[1]) if msg[0] == "ProgramError" else ZeroDivisionError(msg[1])
    st = int(res.status[i])
    return CostModelError(abi.STATUS.get(st, f"status {st}")) if st == 7 else \
        RuntimeError(abi.STATUS.get(st, f"status {st}"))


def evaluate_schedules(program, schedules, arch, launch=None, jobs=None, errors: "list | None" = None) -> list:
    """Drop-in for cmd_rank's evaluate_population over its per-schedule closure
    (apply_schedule + emit_mock_asm + extract_features + score, ls/cli.py:115-121): a list in input
    order of (FeatureVector, score), or None for a failed candidate with (index, exception)
    appended to `errors`.  `jobs` is accepted for API parity (the batch is one device pass)."""
    res = score_batch(program, schedules, arch, launch)
    out = []
    for i in range(len(schedules)):
        if res.status[i]:
            out.append(None)
            if errors is not None:
                errors.append((i, _exception(program, schedules[i], res, i)))
        else:
            out.append((res.feature_vector(i), float(res.scores[i])))
    return out


def optimize(program, space, arch, params, jobs=None, launch=None):
    """Drop-in for es_mod.optimize in cmd_search (ls/cli.py:152): the reference's exact trajectory
    with device-scored generations (es.optimize)."""
    return _optimize(program, space, arch, params, jobs=jobs, launch=launch)


def extract_features(program, code, arch, launch=None, diagnostics=None):
    """Drop-in for cost_mod.extract_features in cmd_analyze (ls/cli.py:89, ls/cost.py:132-152): the
    text-dependent features from the device parser, the IR-side ones from the scoring path."""
    from .code import extract_features as _extract
    return _extract(program, code, arch, launch, diagnostics)

