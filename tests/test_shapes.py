"""Shape generator pins: tensor counts and model sizes of the paper's table
("Characteristics of the benchmark DNN models", "# of
Tensors") and SURVEY.md 8d's configs; cross-checked against HF/torchvision
architectures instantiated on the meta device when those are importable."""
import pytest

from synth import shapes


@pytest.mark.parametrize("model,count,mb", [
    ("vgg16", 32, 528), ("resnet101", 314, 170), ("gpt2_small", 148, 475),
    ("bert_base", 206, 420),   # paper prints 207 tensors; HF BertForPreTraining has 206 unique (tied decoder)
])
def test_paper_model_table(model, count, mb):
    s = shapes.numels(model)
    assert len(s) == count
    assert round(sum(s) * 4 / 2 ** 20) == mb


def test_config_models():
    r50 = shapes.numels("resnet50")
    assert (len(r50), sum(r50), max(r50)) == (161, 25_557_032, 2_359_296)
    assert sum(1 for x in r50 if x < 4096) == 107
    bl = shapes.numels("bert_large")
    assert (len(bl), sum(bl), max(bl)) == (398, 336_226_108, 31_254_528)
    g2 = shapes.numels("gpt2_medium")
    assert (len(g2), sum(g2), max(g2)) == (292, 354_823_168, 51_463_168)
    rule = [shapes.gpt2_medium_mixed_rule(x) for x in g2]
    assert rule.count("dgc") == 49 and rule.count("efsignsgd") == 49 and rule.count("none") == 194


def test_against_transformers_meta():
    transformers = pytest.importorskip("transformers")
    import torch
    with torch.device("meta"):
        m = transformers.BertForPreTraining(transformers.BertConfig(
            hidden_size=1024, num_hidden_layers=24, num_attention_heads=16, intermediate_size=4096))
    assert [p.numel() for p in m.parameters()] == shapes.numels("bert_large")
    with torch.device("meta"):
        m = transformers.GPT2LMHeadModel(transformers.GPT2Config(n_embd=1024, n_layer=24, n_head=16))
    assert [p.numel() for p in m.parameters()] == shapes.numels("gpt2_medium")
