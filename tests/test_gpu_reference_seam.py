"""The documented reference-side seam, exercised with the
REFERENCE ITSELF: the unmodified `metricforge` package installed in
`baseline/_ref` (git-ignored, travels to the GPU box with the snapshot) has
its `ScoringModel` replaced by `GpuScoringModel` at the one place its
`Evaluator` constructs it (`pkg/src/metricforge/evaluate.py:151`). Its own
`Evaluator`, CLI, batching and TSV handling then drive the device path, and
its own CPU `ScoringModel` is the fp32 oracle on the same box.

Checks follow the reference's acceptance suite (`pkg/tests/test_acceptance.py`):
oracle equivalence on the 50-model family (:69-126, ORACLE_TOL 1e-5), batch
composition invariance (:129-156, 1e-6), the fp16 bound (:159-180), the
byte-stable CLI golden (:370-388), and that container errors surface as the
reference's own `metricforge.errors.ContainerError`."""

import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import fixtures as fx

from conftest import ROOT, parity_log, write_model

pytestmark = pytest.mark.gpu

REF = ROOT / "baseline" / "_ref"


@pytest.fixture(scope="module")
def ref():
    if not (REF / "metricforge" / "__init__.py").exists():
        pytest.skip("reference not installed in baseline/_ref (DESIGN.md §7 install command)")
    sys.path.insert(0, str(REF))
    import metricforge
    import metricforge.evaluate as ref_eval

    from paper_2408_11853_b200 import GpuScoringModel
    cpu_model = ref_eval.ScoringModel
    ref_eval.ScoringModel = GpuScoringModel
    yield metricforge, cpu_model
    ref_eval.ScoringModel = cpu_model


def ref_evaluator(mf_ref, fixture_or_path, vocab, **kw):
    return mf_ref.Evaluator(mf_ref.EvaluatorConfig(model=fixture_or_path, vocab=vocab, quiet=True,
                                                   **kw))


def test_reference_evaluator_runs_the_device_model(ref, tiny_qe):
    mf_ref, _ = ref
    from paper_2408_11853_b200 import GpuScoringModel
    with ref_evaluator(mf_ref, tiny_qe.model, tiny_qe.vocab) as ev:
        assert isinstance(ev.model, GpuScoringModel)
        launches0 = ev.model.stats()["kernel_launches"]
        rep = ev.evaluate_lines(fx.fixture_tsv_lines("comet-qe", 20, seed=42))
        assert ev.model.stats()["kernel_launches"] > launches0
    text = "".join(f"{v:.4f}\n" for v in rep.segment_scores)
    assert text == (ROOT / "tests" / "golden" / "eval_qe.txt").read_text()


def test_reference_cli_golden_through_seam(ref, tiny_qe):
    """The reference's own CLI process (`metricforge.cli`), device model patched in."""
    code = ("import sys; import metricforge.evaluate as e; "
            "from paper_2408_11853_b200 import GpuScoringModel; e.ScoringModel = GpuScoringModel; "
            "from metricforge.cli import main; sys.exit(main())")
    env = dict(os.environ, PYTHONPATH=f"{REF}{os.pathsep}{ROOT}")
    tsv = "".join(ln + "\n" for ln in fx.fixture_tsv_lines("comet-qe", 20, seed=42))
    r = subprocess.run([sys.executable, "-c", code, "-m", tiny_qe.model, "-v", tiny_qe.vocab,
                        "--stdin", "--quiet"], input=tsv, capture_output=True, text=True,
                       env=env, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    assert r.stdout == (ROOT / "tests" / "golden" / "eval_qe.txt").read_text()


def test_acceptance_family_vs_reference_cpu_model(ref, tmp_path, vocab_path):
    """test_acceptance.py:69-126 with the reference's own fp32 ScoringModel as
    the oracle (same containers, same encode_fields, same records)."""
    mf_ref, cpu_model = ref
    from metricforge.vocab import encode_fields

    from paper_2408_11853_b200 import GpuScoringModel
    rng = np.random.default_rng(20240917)
    kinds = list(mf_ref.Kind)
    vocab = mf_ref.load_vocab(vocab_path)
    worst = 0.0
    for i in range(50):
        heads = int(rng.choice([1, 2, 4]))
        d = heads * int(rng.choice([4, 8]))
        kind = kinds[i % len(kinds)]
        man = fx.tiny_manifest(kind.value, d_model=d, n_heads=heads,
                               n_layers=int(rng.integers(1, 4)), d_ffn=2 * d, max_position=64,
                               norm_style=str(rng.choice(["pre", "post"])),
                               head_hidden=[[8], [16], [16, 8]][int(rng.integers(0, 3))])
        w = fx.fixture_weights(man, int(rng.integers(0, 2 ** 31)))
        path = write_model(tmp_path / f"m{i}.mfrg", man, w)
        lines = fx.fixture_tsv_lines(kind.value, 20, seed=i)
        with mf_ref.open_container(path) as container:
            records = list(mf_ref.records_from_tsv_lines(lines, kind))
            encoded = [encode_fields(vocab, r, kind, 64) for r in records]
            want = cpu_model(container).score_records(encoded)
            gm = GpuScoringModel(container)
            got = gm.score_records(encoded)
            gm.close()
        worst = max(worst, float(np.abs(got.astype(np.float64) - want).max()))
    parity_log("seam/acceptance_family/50", max_abs=worst)
    assert worst <= 1e-5, worst  # ORACLE_TOL (test_acceptance.py:46)


def test_batch_invariance_through_reference_evaluator(ref, tiny_qe):
    """test_acceptance.py:129-156: sequential vs batched/sorted/4 workers (the
    reference's thread pool calls score_records concurrently)."""
    mf_ref, _ = ref
    lines = fx.fixture_tsv_lines("comet-qe", 1000, seed=314)
    seq_cfg = mf_ref.BatchConfig(mini_batch=1, maxi_batch_factor=1, sort_by_length=False)
    with ref_evaluator(mf_ref, tiny_qe.model, tiny_qe.vocab, batch=seq_cfg) as ev:
        sequential = ev.evaluate_lines(lines).segment_scores
    bat_cfg = mf_ref.BatchConfig(mini_batch=128, maxi_batch_factor=8, sort_by_length=True,
                                 workers=4)
    with ref_evaluator(mf_ref, tiny_qe.model, tiny_qe.vocab, batch=bat_cfg) as ev:
        batched = ev.evaluate_lines(lines).segment_scores
    assert len(sequential) == len(batched) == 1000
    assert sequential == batched  # bitwise; the reference's bound is 1e-6


def test_fp16_bound_through_reference_evaluator(ref, tiny_qe):
    """test_acceptance.py:159-180: the reference's fp16 flag selects the device
    binary16 mode; segment bound 5e-2, system bound 1e-2 against fp32."""
    mf_ref, _ = ref
    lines = fx.fixture_tsv_lines("comet-qe", 200, seed=11)
    out = {}
    for mode in ("fp32", "fp16"):
        with ref_evaluator(mf_ref, tiny_qe.model, tiny_qe.vocab, compute_mode=mode) as ev:
            assert ev.model.precision == mode
            rep = ev.evaluate_lines(lines)
            out[mode] = (rep.segment_scores, rep.system_score)
    seg = max(abs(a - b) for a, b in zip(out["fp32"][0], out["fp16"][0]))
    assert seg <= 5e-2 and abs(out["fp32"][1] - out["fp16"][1]) <= 1e-2


def test_container_errors_are_reference_classes(ref, tmp_path, vocab_path):
    """A mis-shaped tensor raises the reference's ContainerError (`encoder.py:108-115`)."""
    mf_ref, _ = ref
    man = fx.tiny_manifest("comet-qe")
    w = fx.fixture_weights(man, 7)
    w["layer.0.ffn.b1"] = w["layer.0.ffn.b1"][:-1]
    from oracle import mfrg
    path = str(tmp_path / "bad.mfrg")
    shapes = dict(fx.tensor_shapes(man))
    mfrg.write(path, mfrg.manifest_dict(**man), [(n, "f32", w[n]) for n in shapes])
    from metricforge.errors import ContainerError

    from paper_2408_11853_b200 import GpuScoringModel
    with mf_ref.open_container(path, validate=False) as c:
        with pytest.raises(ContainerError, match="ffn.b1"):
            GpuScoringModel(c)
