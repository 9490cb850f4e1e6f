"""Regenerates ddp_buckets.json: DDP gradient-bucket byte sizes (SURVEY.md 8d
config 5) from torch's own bucketing (`_compute_bucket_assignment_by_size`,
caps [1 MiB, 25 MiB], parameters in reverse order, fp32) on ResNet-50
(torchvision, weights=None) and BERT-large (transformers BertForPreTraining,
hidden 1024, 24 layers, 16 heads, intermediate 4096)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def buckets(model):
    from torch._C._distributed_c10d import _compute_bucket_assignment_by_size

    params = list(reversed([p for p in model.parameters() if p.requires_grad]))
    idx, _ = _compute_bucket_assignment_by_size(params, [1 << 20, 25 << 20], [False] * len(params))
    return [sum(params[i].numel() * 4 for i in b) for b in idx]


def models():
    import torchvision
    from transformers import BertConfig, BertForPreTraining

    yield "resnet50", torchvision.models.resnet50(weights=None)
    yield "bert_large", BertForPreTraining(BertConfig(hidden_size=1024, num_hidden_layers=24, num_attention_heads=16,
                                                      intermediate_size=4096))


def main():
    out = {name: buckets(m) for name, m in models()}
    if len(sys.argv) > 1 and sys.argv[1] == "--print":
        print(json.dumps(out))
        return
    json.dump(out, open(os.path.join(ROOT, "tests", "golden", "ddp_buckets.json"), "w"))


if __name__ == "__main__":
    main()
