import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1708_02937_b200 as sk
m, n, kY, L = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), 2
Ws = [sk.gen_layer_fixed(m, 32, sk.layer_seed(17, k), 1.0 / 16) for k in range(L)]
model = sk.DnnModel(Ws, [np.full(m, -0.3, np.float32)] * L)
Y = sk.gen_input_binary(m, n, kY, 17)
if os.environ.get("NOADAPT"): sk.default_context().set_density_switch(0.0, 0.0)
out, tr = sk.relu_forward_sparse(model, Y, sk.ForwardOptions(clip=32.0))
print("trace", list(tr))
