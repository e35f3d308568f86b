"""Command line in the reference's shape (cli.py:334-398 of ``specpipe``), on B200.

    python -m paper_2505_10259_b200 presets [--emit-config NAME]
    python -m paper_2505_10259_b200 pmf P N_CAND
    python -m paper_2505_10259_b200 plan (--config C.json | --preset NAME) [--out DIR] [--simulate-top-k K]
    python -m paper_2505_10259_b200 simulate (--config C.json | --preset NAME) [--policy a,b,c,d]
                                    [--layers L] [--max-rounds R] [--format json|csv|chrome] [--out DIR]

Same config schema (config.py:1-89), output files (``ranking.json``,
``trace.{json,csv,chrome.json}``, ``summary.json``, ``meta.json``) and exit codes
(cli.py:20-30) as the reference; the difference is what ``simulate`` does:
the reference replays its cost model (simulator.py:108-227), this one RUNS the
policy on the GPU (``Engine.run_decoding``: streamed target layers, dual-batch
ping-pong, accept/reject kernels) with synthetic weights of the named shapes
and forced acceptance at the workload's ``acceptance_p`` (T9), and
writes the MEASURED trace.  ``plan --simulate-top-k`` re-ranks the planner's
top k by measured throughput (cli.py:130-157).  ``--layers`` truncates both
models' depth for a quick run (the summary says so).
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import sys
import time

from . import __version__
from .acceptance import AcceptanceModel, expected_accepted, pmf
from .config import arch_for_spec
from .domain import HardwareProfile, ModelSpec, Policy, Workload, validate_profile
from .errors import ConfigError, SpecPipeError, ValidationError

EXIT_OK, EXIT_CONFIG, EXIT_INFEASIBLE, EXIT_INTERNAL = 0, 2, 3, 4
_REQUIRED = ("hardware", "target_model", "draft_model", "workload")
_OPTIONAL = ("policy", "search_space", "seed", "output_dir")


@dataclasses.dataclass
class RunConfig:
    hardware: HardwareProfile
    target_model: ModelSpec
    draft_model: ModelSpec
    workload: Workload
    policy: Policy | None = None
    search_space: object = None
    seed: int = 0
    output_dir: str | None = None

    def to_dict(self) -> dict:
        doc = {"hardware": self.hardware.to_dict(), "target_model": dataclasses.asdict(self.target_model),
               "draft_model": dataclasses.asdict(self.draft_model), "workload": dataclasses.asdict(self.workload),
               "seed": self.seed}
        if self.policy is not None:
            doc["policy"] = dataclasses.asdict(self.policy)
        if self.search_space is not None:
            doc["search_space"] = self.search_space.to_dict()
        return doc


def _typed(cls, data: dict, what: str):
    names = {f.name for f in dataclasses.fields(cls)}
    extra = sorted(set(data) - names)
    if extra:
        raise ConfigError(f"unknown key '{extra[0]}' in {what}")
    return cls(**data)


def parse_config(doc: dict) -> RunConfig:
    """The reference's run-config schema (config.py:49-89), unknown keys rejected."""
    from .planner import SearchSpace

    if not isinstance(doc, dict):
        raise ConfigError("config root must be an object")
    for key in doc:
        if key not in _REQUIRED + _OPTIONAL:
            raise ConfigError(f"unknown key '{key}' at config root")
    for key in _REQUIRED:
        if key not in doc:
            raise ConfigError(f"missing required key '{key}'")
    try:
        return RunConfig(
            hardware=validate_profile(HardwareProfile.from_dict(doc["hardware"])),
            target_model=_typed(ModelSpec, doc["target_model"], "target_model"),
            draft_model=_typed(ModelSpec, doc["draft_model"], "draft_model"),
            workload=_typed(Workload, doc["workload"], "workload"),
            policy=_typed(Policy, doc["policy"], "policy") if "policy" in doc else None,
            search_space=SearchSpace.from_dict(doc["search_space"]) if "search_space" in doc else None,
            seed=int(doc.get("seed", 0)), output_dir=doc.get("output_dir"))
    except ConfigError:
        raise
    except (TypeError, ValueError) as exc:
        raise ConfigError(str(exc)) from exc


def _preset_config(name: str, total_sequences: int = 2 * 192) -> RunConfig:
    from .presets import preset

    hw, target, draft = preset(name)
    return RunConfig(hw, target, draft, Workload(total_sequences=total_sequences, l_input=503, max_new_tokens=16,
                                                 acceptance_p=0.8))


def _load(args) -> RunConfig:
    if getattr(args, "config", None):
        try:
            with open(args.config) as fh:
                doc = json.load(fh)
        except json.JSONDecodeError as exc:
            raise ConfigError(f"invalid JSON in {args.config}: {exc}") from exc
        return parse_config(doc)
    if getattr(args, "preset", None):
        return _preset_config(args.preset)
    raise ConfigError("one of --config or --preset is required")


def _out_dir(args, config: RunConfig) -> str:
    out = args.out or config.output_dir or "specoffload_out"
    os.makedirs(out, exist_ok=True)
    return out


def _write_json(path: str, doc) -> None:
    with open(path, "w") as fh:
        json.dump(doc, fh, indent=2, sort_keys=True)
        fh.write("\n")


def _write_meta(out: str, args, seed: int, extra: dict | None = None) -> None:
    meta = {"version": __version__, "argv": sys.argv[1:], "seed": seed, "config": getattr(args, "config", None),
            "preset": getattr(args, "preset", None), "created_unix": time.time()}
    meta.update(extra or {})
    _write_json(os.path.join(out, "meta.json"), meta)


# ------------------------------------------------------------------ commands

def cmd_presets(args) -> int:
    from .presets import preset, preset_names

    if args.emit_config:
        print(json.dumps(_preset_config(args.emit_config).to_dict(), sort_keys=True, indent=2))
        return EXIT_OK
    for name in preset_names():
        hw, target, draft = preset(name)
        print(f"{name}: target={target.name} ({target.total_bytes() / 1e9:.1f} GB, {target.n_layer} layers), "
              f"draft={draft.name} ({draft.total_bytes() / 1e9:.1f} GB), gpu={hw.gpu_mem_capacity / 1024**3:.0f} GiB")
    return EXIT_OK


def cmd_pmf(args) -> int:
    model = AcceptanceModel(p=args.p, n_cand=args.n_cand)
    print("k\tpmf\tcumulative")
    cum = 0.0
    for k, prob in enumerate(pmf(model), start=1):
        cum += prob
        print(f"{k}\t{prob:.9f}\t{cum:.9f}")
    print(f"expected accepted per round: {expected_accepted(model):.9f}")
    return EXIT_OK


def cmd_plan(args) -> int:
    from . import planner

    config = _load(args)
    out = _out_dir(args, config)
    space = config.search_space or planner.B200_SEARCH_SPACE
    ranked = planner.search(space, config.workload, config.hardware, config.target_model, config.draft_model,
                            strict_paper_approx=args.strict_paper_approx)
    rows = [{"policy": dataclasses.asdict(p), "throughput": round(c.throughput, 6),
             "t_target_per_round": round(c.t_target_per_round, 6), "t_draft_per_round": round(c.t_draft_per_round, 6),
             "v_decoding": c.v_decoding} for p, c in ranked.entries]
    if args.simulate_top_k > 0:  # measure the top k on the GPU (cli.py:130-157)
        for row in rows[: args.simulate_top_k]:
            res, _ = _run(config, Policy(**row["policy"]), args)
            row["measured_throughput"] = round(res.throughput, 6)
        head = sorted(rows[: args.simulate_top_k], key=lambda r: -r["measured_throughput"])
        rows = head + rows[args.simulate_top_k:]
    _write_json(os.path.join(out, "ranking.json"), {"entries": rows, "n_feasible": len(rows)})
    _write_meta(out, args, config.seed)
    best = rows[0]
    print(f"best policy {tuple(best['policy'].values())}: {best.get('measured_throughput', best['throughput']):.3f} "
          f"tok/s ({'measured' if 'measured_throughput' in best else 'predicted'}); {len(rows)} feasible")
    return EXIT_OK


def _archs(config: RunConfig, layers: int):
    t, d = arch_for_spec(config.target_model), arch_for_spec(config.draft_model)
    if t is None or d is None:
        raise ConfigError("simulate runs known architectures only (Mixtral-8x7B/8x22B, Mistral-7B, the tiny pair); "
                          f"got {config.target_model.name!r} / {config.draft_model.name!r}")
    if layers:
        t = dataclasses.replace(t, n_layer=min(layers, t.n_layer))
        d = dataclasses.replace(d, n_layer=min(layers, d.n_layer))
    return t, d


def _run(config: RunConfig, policy: Policy, args):
    """Build a synthetic-weight engine for the config's shapes under its HBM
    budget and run the policy's decode phase on cuda:0."""
    import torch

    from .api import build_engine
    from .engine import Forced
    from .planner_b200 import B200Rates, plan_offload

    t, d = _archs(config, args.layers)
    wl = config.workload
    free = torch.cuda.mem_get_info(0)[0]
    hbm = min(int(config.hardware.gpu_mem_capacity), int(free * 0.92))
    plan = plan_offload(t, d, hbm, int(config.hardware.cpu_mem_capacity), policy.n_cand, wl.acceptance_p,
                        wl.l_input, wl.max_new_tokens, B200Rates(), bs_candidates=[policy.bs_decoding],
                        draft_kv_modes=("cached",))
    eng = build_engine(t, d, device="cuda:0", stream_layers=set(plan.stream_layers), codec="none", trace=True,
                       stream_attn=plan.stream_attn)
    rounds = getattr(args, "max_rounds", 0) or None
    res = eng.run_decoding(policy, dataclasses.replace(wl, total_sequences=2 * policy.bs_decoding),
                           seed=config.seed if args.seed is None else args.seed,
                           acceptance=Forced(wl.acceptance_p), max_rounds=rounds)
    info = {"target": t.name, "draft": d.name, "layers": (t.n_layer, d.n_layer), "streamed_layers": len(plan.stream_layers),
            "hbm_budget_bytes": hbm}
    return res, info


def cmd_simulate(args) -> int:
    from .trace import export_trace

    config = _load(args)
    policy = Policy(*[int(v) for v in args.policy.split(",")]) if args.policy else config.policy
    if policy is None:
        raise ConfigError("'simulate' requires a policy (config key 'policy' or --policy)")
    out = _out_dir(args, config)
    seed = args.seed if args.seed is not None else config.seed
    res, info = _run(config, policy, args)
    ext = {"json": "json", "csv": "csv", "chrome": "chrome.json"}[args.format]
    with open(os.path.join(out, f"trace.{ext}"), "w") as fh:
        fh.write(export_trace(res, args.format))
    busy = {r: round(v / res.total_time, 6) for r, v in res.per_resource_busy.items()} if res.total_time else {}
    _write_json(os.path.join(out, "summary.json"), {
        "policy": dataclasses.asdict(policy), "seed": seed, "total_time_s": round(res.total_time, 6),
        "tokens_generated": res.tokens_generated, "throughput": round(res.throughput, 6),
        "rounds_executed": res.rounds_executed, "peak_gpu_bytes": res.peak_gpu_bytes, "busy_fraction": busy,
        "measured": True, "weights": "synthetic N(0, 0.02^2)", "acceptance": f"forced p={config.workload.acceptance_p}",
        **info})
    _write_meta(out, args, seed, {"measured_on": "cuda:0"})
    print(f"measured {res.tokens_generated} tokens in {res.total_time:.3f} s "
          f"({res.throughput:.3f} tok/s, {res.rounds_executed} rounds)")
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="specoffload-b200",
                                     description="Offloaded speculative decoding on B200 (SpecOffload hot path)")
    parser.add_argument("--version", action="version", version=__version__)
    sub = parser.add_subparsers(dest="command", required=True)

    def source(p):
        g = p.add_mutually_exclusive_group()
        g.add_argument("--config")
        g.add_argument("--preset")

    p_plan = sub.add_parser("plan", help="rank a policy grid by predicted (optionally measured) throughput")
    source(p_plan)
    p_plan.add_argument("--out", default=None)
    p_plan.add_argument("--simulate-top-k", type=int, default=0)
    p_plan.add_argument("--strict-paper-approx", action="store_true")
    p_plan.add_argument("--layers", type=int, default=0, help="truncate model depth for --simulate-top-k runs")
    p_plan.add_argument("--max-rounds", type=int, default=0)
    p_plan.add_argument("--seed", type=int, default=None)
    p_plan.set_defaults(func=cmd_plan)

    p_sim = sub.add_parser("simulate", help="run one policy on the GPU and write its measured trace")
    source(p_sim)
    p_sim.add_argument("--policy", default=None, help="bs_prefill,bs_decoding,bs_draft,n_cand")
    p_sim.add_argument("--out", default=None)
    p_sim.add_argument("--seed", type=int, default=None)
    p_sim.add_argument("--format", choices=["json", "csv", "chrome"], default="json")
    p_sim.add_argument("--layers", type=int, default=0, help="truncate both models to L layers (quick runs)")
    p_sim.add_argument("--max-rounds", type=int, default=0)
    p_sim.set_defaults(func=cmd_simulate)

    p_pmf = sub.add_parser("pmf", help="print the accepted-token distribution")
    p_pmf.add_argument("p", type=float)
    p_pmf.add_argument("n_cand", type=int)
    p_pmf.set_defaults(func=cmd_pmf)

    p_pre = sub.add_parser("presets", help="list built-in B200 presets")
    p_pre.add_argument("--emit-config", default=None, metavar="NAME")
    p_pre.set_defaults(func=cmd_presets)
    return parser


def main(argv: list[str] | None = None) -> int:
    from .errors import InfeasiblePlan, NoFeasiblePolicy

    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except (ConfigError, ValidationError, FileNotFoundError) as exc:
        print(f"config error: {exc}", file=sys.stderr)
        return EXIT_CONFIG
    except NoFeasiblePolicy as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_INFEASIBLE
    except InfeasiblePlan as exc:
        print(f"internal feasibility violation: {exc}", file=sys.stderr)
        return EXIT_INTERNAL
    except SpecPipeError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_CONFIG
