timeout 900 python -m pytest tests/test_mesh_device.py -m gpu -x -q 2>&1 | tail -3
timeout 900 python -c "
import time, numpy as np
from paper_1604_05937_b200.mesh import generate_unit_square_mesh, derive_edges
from paper_1604_05937_b200.ordering import rcm_vertex_order, apply_ordering
import torch; torch.zeros(1).cuda()
t=time.time(); m=generate_unit_square_mesh(2048); t1=time.time(); print('generate 2048 (device edges)', round(t1-t,2))
p=rcm_vertex_order(m); t2=time.time(); print('rcm', round(t2-t1,2))
m2=apply_ordering(m,p); t3=time.time(); print('apply_ordering (device)', round(t3-t2,2))
c=np.asarray(m2.cell_vertices)
t4=time.time(); ev,ce=derive_edges(c, m2.num_vertices, device=True); t5=time.time(); print('derive_edges device', round(t5-t4,3))
ev2,ce2=derive_edges(c, m2.num_vertices, device=False); t6=time.time(); print('derive_edges host', round(t6-t5,2))
print('bit-exact 2048^2:', np.array_equal(ev,ev2) and np.array_equal(ce,ce2))
"
