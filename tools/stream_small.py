"""Small K7 check (for compute-sanitizer): cfg-like layer at a reduced batch,
stream kernel vs the specialised windowed kernel, bitwise."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1708_02937_b200 as sk  # noqa: E402


def main():
    m, B, kY = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    bias = float(sys.argv[4]) if len(sys.argv) > 4 else -0.2
    grp = int(sys.argv[5]) if len(sys.argv) > 5 else 0
    fb = int(sys.argv[6]) if len(sys.argv) > 6 else 0
    ctx = sk.default_context()
    W0 = sk.gen_layer_fixed(m, 32, sk.layer_seed(42, 0), 1.0 / 16)
    Y0 = sk.gen_input_binary(m, B, kY, 42)
    model = sk.DnnModel([W0], [np.full(m, bias, np.float32)])
    opt = sk.ForwardOptions(clip=32.0)
    ctx.set_tuning(exact_kernel=2)
    ref, _ = sk.relu_forward_sparse(model, Y0, opt)
    ctx.set_tuning(exact_kernel=5, exact_group=grp, exact_fields=fb)
    out, _ = sk.relu_forward_sparse(model, Y0, opt)
    print(ctx.last_exact(), ref.nnz(), out.nnz())
    a, b = ref.extract(), out.extract()
    print("same" if all(np.array_equal(x.view(np.uint32), y.view(np.uint32)) for x, y in zip(a, b))
          else "DIFF")


if __name__ == "__main__":
    main()
