"""Synthetic gradient-set shapes (test/bench infrastructure, no method arithmetic).

The paper trains real models (Table "Characteristics of the
benchmark DNN models"; tensor counts in Table "The time to select compression
strategies").  This build has no datasets or weights, so the gradient
set of a model is reproduced from its architecture: one fp32 tensor per
parameter, in `named_parameters()` order, with the exact numel.

Shared by the CUDA path's tests/bench and the oracle: it only describes sizes.
"""
from __future__ import annotations


def _conv(o, i, kh, kw):
    return o * i * kh * kw


def resnet(blocks, bottleneck=True, num_classes=1000):
    """torchvision ResNet parameter numels in registration order."""
    out = [("conv1.weight", _conv(64, 3, 7, 7)), ("bn1.weight", 64), ("bn1.bias", 64)]
    inplanes = 64
    exp = 4 if bottleneck else 1
    for li, (nb, width) in enumerate(zip(blocks, (64, 128, 256, 512))):
        for b in range(nb):
            p = f"layer{li + 1}.{b}."
            if bottleneck:
                out += [(p + "conv1.weight", _conv(width, inplanes, 1, 1)),
                        (p + "bn1.weight", width), (p + "bn1.bias", width),
                        (p + "conv2.weight", _conv(width, width, 3, 3)),
                        (p + "bn2.weight", width), (p + "bn2.bias", width),
                        (p + "conv3.weight", _conv(width * exp, width, 1, 1)),
                        (p + "bn3.weight", width * exp), (p + "bn3.bias", width * exp)]
            else:
                out += [(p + "conv1.weight", _conv(width, inplanes, 3, 3)),
                        (p + "bn1.weight", width), (p + "bn1.bias", width),
                        (p + "conv2.weight", _conv(width, width, 3, 3)),
                        (p + "bn2.weight", width), (p + "bn2.bias", width)]
            if b == 0 and (inplanes != width * exp or li > 0):
                out += [(p + "downsample.0.weight", _conv(width * exp, inplanes, 1, 1)),
                        (p + "downsample.1.weight", width * exp),
                        (p + "downsample.1.bias", width * exp)]
            inplanes = width * exp
    out += [("fc.weight", 512 * exp * num_classes), ("fc.bias", num_classes)]
    return out


def resnet50():
    return resnet((3, 4, 6, 3))


def resnet101():
    return resnet((3, 4, 23, 3))


def vgg16(num_classes=1000):
    cfg = [64, 64, 128, 128, 256, 256, 256, 512, 512, 512, 512, 512, 512]
    out, cin, i = [], 3, 0
    for c in cfg:
        out += [(f"features.{i}.weight", _conv(c, cin, 3, 3)), (f"features.{i}.bias", c)]
        cin, i = c, i + 1
    out += [("classifier.0.weight", 512 * 7 * 7 * 4096), ("classifier.0.bias", 4096),
            ("classifier.3.weight", 4096 * 4096), ("classifier.3.bias", 4096),
            ("classifier.6.weight", 4096 * num_classes), ("classifier.6.bias", num_classes)]
    return out


def bert_pretraining(layers, hidden, inter, vocab=30522, max_pos=512, type_vocab=2):
    """HF BertForPreTraining (decoder weight tied to the word embedding)."""
    h = hidden
    out = [("bert.embeddings.word_embeddings.weight", vocab * h),
           ("bert.embeddings.position_embeddings.weight", max_pos * h),
           ("bert.embeddings.token_type_embeddings.weight", type_vocab * h),
           ("bert.embeddings.LayerNorm.weight", h), ("bert.embeddings.LayerNorm.bias", h)]
    for l in range(layers):
        p = f"bert.encoder.layer.{l}."
        for m in ("query", "key", "value"):
            out += [(p + f"attention.self.{m}.weight", h * h), (p + f"attention.self.{m}.bias", h)]
        out += [(p + "attention.output.dense.weight", h * h), (p + "attention.output.dense.bias", h),
                (p + "attention.output.LayerNorm.weight", h), (p + "attention.output.LayerNorm.bias", h),
                (p + "intermediate.dense.weight", inter * h), (p + "intermediate.dense.bias", inter),
                (p + "output.dense.weight", h * inter), (p + "output.dense.bias", h),
                (p + "output.LayerNorm.weight", h), (p + "output.LayerNorm.bias", h)]
    out += [("bert.pooler.dense.weight", h * h), ("bert.pooler.dense.bias", h),
            ("cls.predictions.bias", vocab),
            ("cls.predictions.transform.dense.weight", h * h),
            ("cls.predictions.transform.dense.bias", h),
            ("cls.predictions.transform.LayerNorm.weight", h),
            ("cls.predictions.transform.LayerNorm.bias", h),
            ("cls.seq_relationship.weight", 2 * h), ("cls.seq_relationship.bias", 2)]
    return out


def bert_large():
    return bert_pretraining(24, 1024, 4096)


def bert_base():
    return bert_pretraining(12, 768, 3072)


def gpt2(layers, d, vocab=50257, n_pos=1024):
    """HF GPT2LMHeadModel (lm_head tied to wte)."""
    out = [("transformer.wte.weight", vocab * d), ("transformer.wpe.weight", n_pos * d)]
    for l in range(layers):
        p = f"transformer.h.{l}."
        out += [(p + "ln_1.weight", d), (p + "ln_1.bias", d),
                (p + "attn.c_attn.weight", d * 3 * d), (p + "attn.c_attn.bias", 3 * d),
                (p + "attn.c_proj.weight", d * d), (p + "attn.c_proj.bias", d),
                (p + "ln_2.weight", d), (p + "ln_2.bias", d),
                (p + "mlp.c_fc.weight", d * 4 * d), (p + "mlp.c_fc.bias", 4 * d),
                (p + "mlp.c_proj.weight", 4 * d * d), (p + "mlp.c_proj.bias", d)]
    out += [("transformer.ln_f.weight", d), ("transformer.ln_f.bias", d)]
    return out


def gpt2_small():
    return gpt2(12, 768)


def gpt2_medium():
    return gpt2(24, 1024)


MODELS = {
    "resnet50": resnet50, "resnet101": resnet101, "vgg16": vgg16,
    "bert_large": bert_large, "bert_base": bert_base,
    "gpt2_small": gpt2_small, "gpt2_medium": gpt2_medium,
}


def numels(model: str):
    return [n for _, n in MODELS[model]()]


def gpt2_medium_mixed_rule(numel: int) -> str:
    """Config 5's fixed strategy rule: N >= 2^22 -> DGC 1% Allgather;
    2^20 <= N < 2^22 -> EFSignSGD Alltoall/Allgather; else NONE Allreduce."""
    if numel >= 1 << 22:
        return "dgc"
    if numel >= 1 << 20:
        return "efsignsgd"
    return "none"
