"""Generate the robot's self-collision pair list -- run once, output pasted into
workloads/scenes.py as data.  Calls only oracle/ (forward kinematics).

Rule (the usual "disabled collision pairs" of motion planners): check sphere pairs on links that are not
adjacent (|link_i - link_j| >= 2) and that do not overlap in more than 90 % of uniformly sampled joint
configurations (structural overlaps of the sphere model, e.g. around the spherical wrist)."""
import numpy as np
import torch

from oracle import tamp_oracle as O
from workloads import panda_robot

r = panda_robot()
rng = np.random.default_rng(0)
q = rng.uniform(r.joint_lo, r.joint_hi, (4000, 7))
W = O.robot_sphere_centers(r, O.forward_kinematics(r, torch.tensor(q))).numpy()
rad, L = r.spheres[:, 3], r.sphere_link
pairs = []
for i in range(len(rad)):
    for j in range(i + 1, len(rad)):
        if abs(int(L[i]) - int(L[j])) < 2:
            continue
        hit = (np.linalg.norm(W[:, i] - W[:, j], axis=-1) < rad[i] + rad[j]).mean()
        if hit <= 0.9:
            pairs.append((i, j))
print(len(pairs))
print(pairs)
