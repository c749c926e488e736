"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the reference package ``ucp`` from /root/reference/pkg/src and
records, for later comparison on machines without the reference:

* generator bit patterns (reference test FROZEN table + extra windows),
* bf16 / f16 cast tables over special values and 2^14 random bit patterns,
* partial-noise tables for tp in {2,3,4,5,8}, every rank,
* per-(spec, cfg) digests of ``enumerate_rank_records`` for every rank,
* whole-pipeline digests (source tree, atomic tree, loaded world in F32,
  BF16 and F16) for a grid of (family, source cfg, target cfg) cells,
* model.json dicts of the specs used, and golden_vec16.ucpt (reference
  test criterion 7, whose fixture is absent from the mount).

Nothing here is imported by the product; the outputs are small data files.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import ucp  # noqa: E402
from ucp import DType, ParallelConfig, PPSchedule, ZeroStage  # noqa: E402
from ucp.models import spec_to_dict  # noqa: E402
from ucp.parallel import enumerate_rank_records, partial_noise  # noqa: E402
from ucp.tensor import cast, gen_tensor, hash_unit, make_tensor, stream_base, write_tensor  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def cfg(dp=1, tp=1, pp=1, sp=1, zero="z0", v=0):
    sched = PPSchedule("interleaved", v) if v else PPSchedule()
    return ParallelConfig(dp=dp, tp=tp, pp=pp, sp=sp, zero_stage=ZeroStage(zero), pp_schedule=sched)


def cfg_key(c) -> str:
    return ucp.format_config_string(c)


def rec_json(r) -> list:
    return [r.param, r.kind, r.pattern, list(r.placement), list(r.shape),
            None if r.segments is None else [list(s) for s in r.segments],
            None if r.flat_range is None else list(r.flat_range), r.pad_elems]


def dir_digest(root: str) -> str:
    h = hashlib.sha256()
    for dirpath, dirnames, filenames in os.walk(root):
        dirnames.sort()
        for name in sorted(filenames):
            p = os.path.join(dirpath, name)
            h.update(os.path.relpath(p, root).encode())
            h.update(b"\0")
            with open(p, "rb") as f:
                h.update(f.read())
            h.update(b"\1")
    return h.hexdigest()


def world_digest(world) -> str:
    h = hashlib.sha256()
    for g in sorted(world.shards):
        for s in world.shards[g]:
            t = s.tensor
            h.update(f"{g}|{s.meta.param}|{s.meta.kind}|{t.dtype.name}|{t.shape}".encode())
            h.update(np.ascontiguousarray(t.data).tobytes())
    return h.hexdigest()


SCALES = {
    "DenseGPT": {"n_layers": 4, "hidden": 64},
    "MoE": {"n_layers": 4, "hidden": 64, "n_experts": 4},
    "GQA": {"n_layers": 4, "hidden": 64, "q_heads": 8, "kv_heads": 2},
}

# (name, family, scale, src cfg, tgt cfg)
PIPELINES = [
    ("cfg1", "DenseGPT", {"n_layers": 12, "hidden": 768}, cfg(2, 2, 2, zero="z1"), cfg(4, zero="z1")),
    ("pad", "DenseGPT", {"n_layers": 2, "hidden": 32}, cfg(3, zero="z3"), cfg(3, 2, zero="z1")),
    ("gqa", "GQA", SCALES["GQA"], cfg(2, 2, 2, zero="z1"), cfg(2, 4, zero="z1")),
    ("moe", "MoE", SCALES["MoE"], cfg(1, 2, 2), cfg(2, 4, zero="z1")),
]
GRID_CFGS = [
    cfg(), cfg(2), cfg(2, zero="z1"), cfg(3, zero="z3"), cfg(4, zero="z3"),
    cfg(1, 2), cfg(2, 2, zero="z1"), cfg(1, 4, 2), cfg(2, 2, 2, zero="z1"),
    cfg(1, 1, 4), cfg(2, 1, 2, zero="z1", v=2), cfg(4, 2, sp=2, zero="z1"),
    cfg(1, 8), cfg(3, 2, zero="z1"), cfg(2, 4, 4, zero="z1"),
]
# reshard cells over the small families: src -> tgt
GRID_PAIRS = [
    (cfg(2, 2, 2, zero="z1"), cfg(4, zero="z1")),
    (cfg(3, zero="z3"), cfg(1, 2, 2)),
    (cfg(1, 4, 2), cfg(2, 2, zero="z1")),
    (cfg(2, 1, 2, zero="z1", v=2), cfg(3, 2, zero="z1")),
    (cfg(4, zero="z3"), cfg(2, 8, zero="z1")),
    (cfg(1, 2), cfg(4, 2, sp=2, zero="z1")),
]


def main() -> None:
    out: dict = {"reference": "/root/reference/pkg/src/ucp", "numpy": np.__version__}
    arrays: dict = {}

    # --- generator ---------------------------------------------------------
    gens = []
    for seed, name, tag, start, count in [
        (7, "layers.0.attn_qkv", "weight", 0, 64), (7, "layers.0.attn_qkv", "m", 0, 64),
        (0, "embed.tokens", "weight", 0, 64), (123456789, "pos.alibi", "v", 0, 64),
        (7, "embed.tokens", "weight", 1_000_000, 256), (2**64 - 1, "x", "grad.3", 77, 100),
        (7, "layers.31.mlp_down", "v", (1 << 32) - 50, 100),
    ]:
        base = stream_base(seed, name, tag)
        vals = hash_unit(base, start, count)
        gens.append({"seed": seed, "name": name, "tag": tag, "start": start, "base": base,
                     "bits": [int(x) for x in vals.view(np.uint32)]})
    out["generator"] = gens

    # --- casts -----------------------------------------------------------------
    rng = np.random.default_rng(20261017)
    special = np.array([
        0x00000000, 0x80000000, 0x7F800000, 0xFF800000, 0x7FC00001, 0x7F800001, 0xFFA00000,
        0x7F7FFFFF, 0x477FF000, 0x477FE000, 0x33000000, 0x33000001, 0x387FC000, 0x38800000,
        0x3F800001, 0x3F808000, 0x3F818000, 0x00008000, 0x00000001, 0x807FFFFF, 0x3F7FFFFF,
        0x3FFFFFFF, 0x7FFFFFFF, 0xFFFFFFFF, 0x38000000, 0x37FFFFFF, 0x33800000, 0x337FFFFF,
    ], dtype=np.uint32)
    bits = np.concatenate([special, rng.integers(0, 2**32, size=1 << 14, dtype=np.uint64).astype(np.uint32)])
    x = bits.view(np.float32)
    arrays["cast_in"] = bits
    arrays["cast_bf16"] = cast(make_tensor(DType.F32, x), DType.BF16).data.astype(np.uint16)
    with np.errstate(all="ignore"):
        arrays["cast_f16"] = cast(make_tensor(DType.F32, x), DType.F16).data.view(np.uint16)

    # --- partial noise -----------------------------------------------------------
    nz_bits = np.concatenate([
        special, rng.integers(0, 2**32, size=4096, dtype=np.uint64).astype(np.uint32),
        np.arange(0, 64, dtype=np.uint32), 0x80000000 + np.arange(0, 64, dtype=np.uint32),
        0x7F7FFFF0 + np.arange(0, 16, dtype=np.uint32), 0x3F7FFFF8 + np.arange(0, 16, dtype=np.uint32),
    ])
    arrays["noise_in"] = nz_bits
    for tp in (2, 3, 4, 5, 8):
        for t in range(tp):
            with np.errstate(all="ignore"):
                arrays[f"noise_tp{tp}_r{t}"] = partial_noise(nz_bits.view(np.float32), t, tp).view(np.uint32)

    # --- models + records ----------------------------------------------------------
    specs = {fam: ucp.make_model(fam, sc) for fam, sc in SCALES.items()}
    for name, fam, sc, _, _ in PIPELINES:
        specs[name] = ucp.make_model(fam, sc)
    specs["dense_l0_h16"] = ucp.make_model("DenseGPT", {"n_layers": 0, "hidden": 16})
    specs["dense_l0_h1024"] = ucp.make_model("DenseGPT", {"n_layers": 0, "hidden": 1024})
    out["models"] = {k: spec_to_dict(s) for k, s in specs.items()}
    recs = {}
    for fam in SCALES:
        for c in GRID_CFGS:
            try:
                ucp.parallel.validate_model_config(specs[fam], c)
            except ucp.UcpError as e:
                recs[f"{fam}|{cfg_key(c)}"] = {"error": type(e).__name__}
                continue
            allr = [[rec_json(r) for r in enumerate_rank_records(specs[fam], c, g)]
                    for g in range(c.world_size)]
            recs[f"{fam}|{cfg_key(c)}"] = {
                "sha256": hashlib.sha256(json.dumps(allr).encode()).hexdigest(),
                "n": sum(len(r) for r in allr)}
    out["records"] = recs

    # --- pipelines -----------------------------------------------------------------
    pipes = []
    cells = [(n, specs[n], s, t) for n, _, _, s, t in PIPELINES]
    for fam in SCALES:
        for i, (s, t) in enumerate(GRID_PAIRS):
            cells.append((f"{fam}.{i}", specs[fam], s, t))
    with tempfile.TemporaryDirectory() as tmp:
        for name, spec, s, t in cells:
            state = ucp.init_state(spec, 7)
            src = os.path.join(tmp, name + "_src")
            atom = os.path.join(tmp, name + "_atomic")
            ucp.partition(state, s, src)
            ucp.convert(src, atom)
            row = {"name": name, "model": spec.name, "src": cfg_key(s), "tgt": cfg_key(t),
                   "src_digest": dir_digest(src), "atomic_digest": dir_digest(atom)}
            for dt in (DType.F32, DType.BF16, DType.F16):
                with np.errstate(all="ignore"):
                    w = ucp.load(atom, t, dtype=dt)
                row[f"world_{dt.name}"] = world_digest(w)
                if dt is DType.F32:
                    row["stats"] = {k: v for k, v in w.stats.to_dict().items() if k != "per_rank"}
            pipes.append(row)
            print("pipeline", name, row["atomic_digest"][:12], flush=True)
        # criterion-7 vector
        write_tensor(os.path.join(HERE, "golden_vec16.ucpt"), gen_tensor(7, "pos.alibi", "weight", (16,)))
        root = os.path.join(tmp, "c7")
        ucp.partition(ucp.init_state(specs["dense_l0_h16"], 7), cfg(), root)
        out["golden_shards_sha256"] = hashlib.sha256(
            open(os.path.join(root, "rank_0", "shards.json"), "rb").read()).hexdigest()
    out["pipelines"] = pipes

    # --- the reference's own verification grid (ucp/verify.py:301-357): 117
    # identity cells (39 configs x 3 stock models) + 21 cross-config cells
    from ucp.verify import resume_pairs, roundtrip_configs, stock_models

    grid = []
    with tempfile.TemporaryDirectory() as tmp:
        cells = [(fam, c, c) for fam, _ in stock_models() for c in roundtrip_configs()]
        cells += [(fam, a, b) for fam, _ in stock_models() for a, b in resume_pairs()]
        for k, (fam, a, b) in enumerate(cells):
            spec = specs[fam]
            state = ucp.init_state(spec, 11)
            src = os.path.join(tmp, f"s{k}")
            atom = os.path.join(tmp, f"a{k}")
            ucp.partition(state, a, src)
            ucp.convert(src, atom)
            row = {"model": fam, "src": cfg_key(a), "tgt": cfg_key(b),
                   "src_digest": dir_digest(src), "atomic_digest": dir_digest(atom)}
            for dt in (DType.F32, DType.BF16):
                row[f"world_{dt.name}"] = world_digest(ucp.load(atom, b, dtype=dt))
            grid.append(row)
    out["grid"] = grid
    print("grid cells", len(grid))

    # --- toy trainer (ucp/models.py:247-328): trained-state digests
    from ucp.models import TrainerConfig, train_steps

    def state_digest(st) -> str:
        h = hashlib.sha256()
        for p in st.spec.params:
            for kind in ("weight", "m", "v"):
                h.update(f"{p.name}|{kind}|".encode())
                h.update(np.ascontiguousarray(getattr(st.params[p.name], kind).data).tobytes())
        h.update(f"step={st.step}".encode())
        return h.hexdigest()

    trained = []
    for fam in SCALES:
        for n in (1, 3):
            st = train_steps(ucp.init_state(specs[fam], 7), TrainerConfig(), 0, n)
            trained.append({"model": fam, "steps": n, "digest": state_digest(st),
                            "iteration": st.metadata["iteration"]})
    st = train_steps(ucp.init_state(specs["GQA"], 7), TrainerConfig(lr=3e-2, beta1=0.8, grad_seed=5),
                     0, 4)
    trained.append({"model": "GQA", "steps": 4, "cfg": {"lr": 3e-2, "beta1": 0.8, "grad_seed": 5},
                    "digest": state_digest(st), "iteration": 4})
    out["trained"] = trained

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
        f.write("\n")
    np.savez_compressed(os.path.join(HERE, "golden_arrays.npz"), **arrays)
    print("wrote", len(pipes), "pipelines,", len(recs), "record sets")


if __name__ == "__main__":
    main()
