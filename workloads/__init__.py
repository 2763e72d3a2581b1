"""Seeded synthetic workloads shared by the oracle and the CUDA path.

This package holds *inputs only*: robot/scene constants and plan skeletons
(Appendix B of SURVEY.md, all PROPOSAL -- the paper publishes no robot model
or scene files).  It contains none of the method's arithmetic (no FK, no
costs, no samplers); the oracle (`oracle/`) and the product library
(`paper_2411_11833_b200/`) each interpret these specs independently.
"""
from .scenes import (  # noqa: F401
    ProblemSpec, Robot, OBB, Obj, Surface, Var, Action,
    CONF, PLACEMENT, GRASP, TRAJ,
    MOVE_FREE, PICK, MOVE_HOLD, PLACE,
    panda_robot, make_config, CONFIG_NAMES, CONFIG_SIZES,
)
